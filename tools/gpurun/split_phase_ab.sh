# Split phases (delivery warps run ahead, no grid barrier): parity with VXB_SPLIT_PHASES=1, then A/B.
export VXB_SPLIT_PHASES=1
timeout 300 python -m pytest tests/test_engine_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_sp.log 2>&1; echo pytest_engine=$?; tail -3 gpurun_out/pytest_sp.log
timeout 600 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "not noise" > gpurun_out/pytest_sp_all.log 2>&1; echo pytest_all=$?; tail -3 gpurun_out/pytest_sp_all.log
for rep in 1 2; do for sp in 0 1; do
VXB_SPLIT_PHASES=$sp timeout 120 python tools/decompose.py config2 --steps 100 --reps 3 > gpurun_out/sp_$sp.log 2>&1; echo "c2 split=$sp rc=$? $(tail -1 gpurun_out/sp_$sp.log | cut -c1-160)"; done; done
for sp in 0 1; do VXB_SPLIT_PHASES=$sp timeout 300 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/sp3_$sp.log 2>&1; echo "c3 split=$sp rc=$? $(tail -1 gpurun_out/sp3_$sp.log | cut -c1-60)"; done
