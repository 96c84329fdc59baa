ts() { date +%T; }
echo "$(ts) tests"; timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE > gpurun_out/g4b_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/g4b_tests.log
echo "$(ts) c2"; timeout 1200 python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu > gpurun_out/g4b_c2.log 2>&1; echo rc=$?
grep '^{' gpurun_out/g4b_c2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','exposed_exchange_us_per_step','exchange_arrival_lag_us_per_step']})"
echo "$(ts) c2 n2"; timeout 1200 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/g4b_c2n2.log 2>&1; echo rc=$?
grep '^{' gpurun_out/g4b_c2n2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','exposed_exchange_us_per_step','exchange_arrival_lag_us_per_step']})"
echo "$(ts) done"
