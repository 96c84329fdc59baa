# config 3 / 5 at 4 GPUs: static deal block-major (new default) vs list-major (round 1)
for w in config3 config5; do for lm in 0 1; do
VXB_TUNING=1 VXB_STATIC_LIST_MAJOR=$lm timeout 2400 python bench.py --gpus 4 --workload $w --steps 3 --warmup 2 --no-cpu > gpurun_out/c5m.log 2>&1
echo "$w list_major=$lm $(grep '^{' gpurun_out/c5m.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(d.get(k),3) for k in ['value','ms_per_step','wall_s_per_bio_s','exposed_exchange_us_per_step']}, d['config']['schedule'].get('static_block_major'))")"
done; done
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE 2>&1 | tail -2
