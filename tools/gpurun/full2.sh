# one GPU: full pytest -m gpu, smoke, phase profile, bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1 || { tail -20 gpurun_out/f_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rfE > gpurun_out/f_tests.log 2>&1; echo tests_rc=$?
tail -8 gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/f_smoke.log
timeout 600 python tools/phase_profile.py --steps 50 --reps 2 2>&1 | grep -E "phase profile|advance" | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.log 2>&1; echo bench_rc=$?
grep '^{' gpurun_out/f_bench.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','e2e','roofline']})"
