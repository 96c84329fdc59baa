# Runtime stage size: config 3 at 768 vs 1024 (default for L2-blocked), config 2 at 768 (default) vs 1024; parity subset.
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "not noise and not multigpu" > gpurun_out/pytest_se.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_se.log
for rep in 1 2; do for e in 768 1024; do
VXB_STAGE_ENTRIES=$e timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz > gpurun_out/se2_$e.log 2>&1; echo "c2 se=$e $(tail -1 gpurun_out/se2_$e.log | cut -c1-50)"; done; done
for e in 768 1024; do VXB_STAGE_ENTRIES=$e timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/se3_$e.log 2>&1; echo "c3 se=$e $(tail -1 gpurun_out/se3_$e.log | cut -c1-50)"; done
