timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE 2>&1 | tail -2
for n in 4; do timeout 2400 python bench.py --gpus $n --workload config5 --steps 5 --warmup 2 --no-cpu > gpurun_out/c5f.log 2>&1
grep '^{' gpurun_out/c5f.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['config']['schedule']; print({k:round(d.get(k),3) for k in ['value','ms_per_step','exposed_exchange_us_per_step']}, s.get('l2_blocks'), s.get('dynamic_deal'))"; done
