# config 5 at 4 GPUs: L2 block size (passes per phase) and deal
for cfg in "VXB_BLOCK_MB=400" "VXB_BLOCK_MB=160" "VXB_BLOCK_MB=400 VXB_DYN=1"; do
env VXB_TUNING=1 $cfg timeout 2400 python bench.py --gpus 4 --workload config5 --steps 3 --warmup 2 --no-cpu > gpurun_out/c5b.log 2>&1
echo "$cfg $(grep '^{' gpurun_out/c5b.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['config']['schedule']; print({k:round(d.get(k),3) for k in ['value','ms_per_step','exposed_exchange_us_per_step']}, s.get('l2_blocks'), s.get('dynamic_deal'))")"
done
