# one GPU: selected tests (PYTEST_SEL) + the default bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1 || { tail -20 gpurun_out/q_build.log; exit 1; }
timeout 1800 python -m pytest -q -p no:cacheprovider -rfE ${PYTEST_SEL} > gpurun_out/q_tests.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/q_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/q_bench.log 2>&1; echo bench_rc=$?
grep '^{' gpurun_out/q_bench.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','e2e','roofline','cpu_baseline']})"
