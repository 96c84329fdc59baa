for cfg in "config5 VXB_BLOCK_MB=210" "config5 VXB_BLOCK_MB=110" "config3 VXB_BLOCK_MB=100" "config3 VXB_BLOCK_MB=64"; do
set -- $cfg; w=$1; shift
env VXB_TUNING=1 "$@" timeout 2400 python bench.py --gpus 4 --workload $w --steps 3 --warmup 2 --no-cpu > gpurun_out/c5c.log 2>&1
echo "$cfg $(grep '^{' gpurun_out/c5c.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['config']['schedule']; print({k:round(d.get(k),3) for k in ['value','ms_per_step','exposed_exchange_us_per_step']}, s.get('l2_blocks'), s.get('dynamic_deal'))")"
done
