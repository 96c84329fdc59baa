# Partial L2 residency of the update state on config 3 (L2-blocked): VXB_FKEEP neurons kept evict_last.
VXB_FKEEP=2000000 timeout 600 python -m pytest tests/test_fullsize_gpu.py -q -p no:cacheprovider -x > gpurun_out/pytest_fkeep.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_fkeep.log
for rep in 1 2; do for fk in 0 500000 1000000 2000000 4000000; do
VXB_FKEEP=$fk timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/fkeep_$fk.log 2>&1; echo "c3 fkeep=$fk $(tail -1 gpurun_out/fkeep_$fk.log | cut -c1-80)"; done; done
