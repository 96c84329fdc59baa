# ensemble members together vs serial + the ensemble tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1 || { tail -20 gpurun_out/e_build.log; exit 1; }
timeout 900 python -m pytest tests/test_ensemble_gpu.py -q -p no:cacheprovider -rfE 2>&1 | tail -3
for v in 100 10; do for p in l2 tile; do timeout 600 python tools/ensemble_batch.py --members 8 --voxels $v --path $p 2>&1 | tail -1; done; done
