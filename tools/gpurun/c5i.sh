timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE 2>&1 | tail -1
timeout 2400 python bench.py --gpus 4 --workload config5 --steps 5 --warmup 2 --no-cpu > gpurun_out/c5i.log 2>&1
grep '^{' gpurun_out/c5i.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['config']['schedule']; print({k:round(d.get(k),3) for k in ['value','ms_per_step','exposed_exchange_us_per_step']}, s.get('l2_blocks'), s.get('dynamic_deal'))"
timeout 2400 python bench.py --gpus 4 --workload config3 --steps 5 --warmup 2 --no-cpu > gpurun_out/c3i.log 2>&1
grep '^{' gpurun_out/c3i.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['config']['schedule']; print({k:round(d.get(k),3) for k in ['value','ms_per_step','exposed_exchange_us_per_step']}, s.get('l2_blocks'), s.get('dynamic_deal'))"
