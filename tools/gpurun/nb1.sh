# barrier-free tile kernel: phase profile, tests, bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/nb_build.log 2>&1 || { tail -20 gpurun_out/nb_build.log; exit 1; }
timeout 300 python tools/phase_profile.py --steps 50 --reps 2 2>&1 | grep -E "phase profile|advance" | tail -3
timeout 1200 python -m pytest -x -q -p no:cacheprovider -rfE -m gpu tests > gpurun_out/nb_tests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/nb_tests.log
timeout 600 python bench.py > gpurun_out/nb_bench.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/nb_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','ms_per_step')}, d['e2e']['value'], d['roofline']['frac'])"
