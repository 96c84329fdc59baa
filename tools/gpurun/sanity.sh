timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_s2.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_s2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s2.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_s2.log
python bench.py > gpurun_out/bench_s2.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_s2.log
