# two GPUs: multi-GPU parity (both paths), abort test, bench --gpus 2 both paths, phase profile
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1 || { tail -20 gpurun_out/m_build.log; exit 1; }
timeout 900 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE > gpurun_out/m_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/m_tests.log
for p in tile l2; do
  VXB_TUNING=1 VXB_PATH=$p timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 tests/dist_check.py > gpurun_out/m_dist_$p.log 2>&1; echo dist_${p}_rc=$?; grep '^{' gpurun_out/m_dist_$p.log | tail -1 | cut -c1-300
  VXB_TUNING=1 VXB_PATH=$p timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/m_bench2_$p.log 2>&1; echo bench2_${p}_rc=$?
  grep '^{' gpurun_out/m_bench2_$p.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','exposed_exchange_us_per_step','e2e']})"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 tools/phase_profile.py --steps 50 --reps 2 2>&1 | grep -E "phase profile|advance" | tail -4
