set -x
nvidia-smi -L; free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g1_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g1_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/g1_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g1_bench.log 2>&1; echo bench_rc=$?
tail -2 gpurun_out/g1_bench.log
