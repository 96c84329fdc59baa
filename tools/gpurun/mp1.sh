# multi-pass tile path: parity tests, then config 3 / config 5 shapes on one GPU
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mp_build.log 2>&1 || { tail -20 gpurun_out/mp_build.log; exit 1; }
timeout 1500 python -m pytest -x -q -p no:cacheprovider -rfE -k "mp or multipass or criterion9" tests/test_engine_gpu.py tests/test_headline_parity_gpu.py tests/test_timings_gpu.py > gpurun_out/mp_tests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/mp_tests.log
summ() { grep '^{' $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','wall_s_per_bio_s','mean_rate_hz','device_memory_used_gb']}, d['config']['schedule'])"; }
timeout 1800 python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu > gpurun_out/mp_c3.log 2>&1; echo rc=$?; summ gpurun_out/mp_c3.log
