for cfg in "VXB_BLOCK_MB=64" "VXB_BLOCK_MB=110" "VXB_BLOCK_MB=160"; do
env VXB_TUNING=1 $cfg timeout 2400 python bench.py --workload config3 --steps 5 --warmup 2 --no-cpu > gpurun_out/c3d.log 2>&1
echo "1gpu c3 $cfg $(grep '^{' gpurun_out/c3d.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['config']['schedule']; print({k:round(d.get(k),3) for k in ['value','ms_per_step']}, s.get('l2_blocks'), s.get('dynamic_deal'))")"
done
