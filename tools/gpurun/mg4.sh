# four GPUs: multi-GPU tests, then config 2 / 3 / 5 lines (bench --gpus 4)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g4_build.log 2>&1 || { tail -20 gpurun_out/g4_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE > gpurun_out/g4_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/g4_tests.log
summ() { grep '^{' $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','wall_s_per_bio_s','mean_rate_hz','exposed_exchange_us_per_step','exchange_arrival_lag_us_per_step','device_memory_used_gb']}, d['config']['schedule']['path'], d['config']['schedule'].get('l2_blocks'))"; }
for w in ${WORKLOADS:-config2 config3 config5}; do
  timeout 1800 python bench.py --gpus 4 --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu > gpurun_out/g4_$w.log 2>&1; echo "$w rc=$?"; summ gpurun_out/g4_$w.log
done
