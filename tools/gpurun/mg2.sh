# two GPUs: multi-GPU parity (tile path and l2 path), abort, full-size 2 == 1, bench --gpus 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1 || { tail -20 gpurun_out/m_build.log; exit 1; }
nvidia-smi topo -m | head -5
timeout 1800 python -m pytest tests/test_multigpu.py tests/test_timings_gpu.py tests/test_ensemble_gpu.py -q -p no:cacheprovider -rfE > gpurun_out/m_tests.log 2>&1; echo tests_rc=$?
tail -8 gpurun_out/m_tests.log
for p in tile l2; do
  VXB_TUNING=1 VXB_PATH=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 tests/dist_check.py > gpurun_out/m_dist_$p.log 2>&1; echo dist_${p}_rc=$?; grep '^{' gpurun_out/m_dist_$p.log | tail -1 | cut -c1-400
done
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/m_bench2.log 2>&1; echo bench2_rc=$?
grep '^{' gpurun_out/m_bench2.log | tail -1 | cut -c1-900
