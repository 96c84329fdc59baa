# multi-pass tile path: parity tests + config 3 phase profile (tile_mp vs l2)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mp_build.log 2>&1 || { tail -20 gpurun_out/mp_build.log; exit 1; }
timeout 1500 python -m pytest -x -q -p no:cacheprovider -rfE -k "mp or multipass or criterion9" tests/test_engine_gpu.py tests/test_headline_parity_gpu.py tests/test_timings_gpu.py > gpurun_out/mp_tests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/mp_tests.log
timeout 900 python tools/phase_profile.py --workload config3 --steps 10 --reps 2 2>&1 | grep -E "phase profile|advance|path" | tail -3
VXB_TILE_ITEMS=0 timeout 900 python tools/phase_profile.py --workload config3 --steps 10 --reps 2 2>&1 | grep -E "phase profile|advance" | tail -2
timeout 900 python tools/phase_profile.py --workload config3 --steps 10 --reps 2 --path l2 2>&1 | grep -E "phase profile|advance" | tail -2
