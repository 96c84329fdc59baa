for w in config3 config5; do for bm in b200 b200_time; do
timeout 2400 python bench.py --gpus 4 --workload $w --byte-model $bm --steps 3 --warmup 2 --no-cpu > gpurun_out/bt4.log 2>&1
echo "$w $bm $(grep '^{' gpurun_out/bt4.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(d.get(k),3) for k in ['value','ms_per_step','exposed_exchange_us_per_step','device_memory_used_gb']})")"
done; done
