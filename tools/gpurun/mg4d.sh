for n in 4 2; do
timeout 1200 python bench.py --gpus $n --steps 20 --warmup 3 --no-cpu > gpurun_out/g4d.log 2>&1
echo "n=$n $(grep '^{' gpurun_out/g4d.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(d.get(k),3) for k in ['value','ms_per_step','exposed_exchange_us_per_step','exchange_arrival_lag_us_per_step']})")"
done
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE 2>&1 | tail -2
