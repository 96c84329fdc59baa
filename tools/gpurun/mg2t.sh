# two GPUs at HEAD: multi-GPU tests, dist parity (tile, l2), bench --gpus 2 (timestamps)
ts() { date +%T; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m2_build.log 2>&1 || { tail -20 gpurun_out/m2_build.log; exit 1; }
echo "$(ts) tests"; timeout 1500 python -m pytest tests/test_multigpu.py tests/test_timings_gpu.py tests/test_ensemble_gpu.py -q -p no:cacheprovider -rfE > gpurun_out/m2_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/m2_tests.log
for p in tile l2; do
  echo "$(ts) dist $p"; VXB_TUNING=1 VXB_PATH=$p timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 tests/dist_check.py > gpurun_out/m2_dist_$p.log 2>&1; echo dist_${p}_rc=$?; grep '^{' gpurun_out/m2_dist_$p.log | tail -1 | cut -c1-200
done
echo "$(ts) bench2"; timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/m2_bench2.log 2>&1; echo bench2_rc=$?
grep '^{' gpurun_out/m2_bench2.log | tail -1 | cut -c1-300
echo "$(ts) done"
