# two GPUs: bench --gpus 2 on both paths + tile-path phase profile per rank
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1 || { tail -20 gpurun_out/m_build.log; exit 1; }
for p in tile l2; do
  VXB_TUNING=1 VXB_PATH=$p timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu > gpurun_out/m_bench2_$p.log 2>&1; echo bench2_${p}_rc=$?
  grep '^{' gpurun_out/m_bench2_$p.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','ms_per_step','exposed_exchange_us_per_step','e2e']})"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29541 tools/phase_profile.py --steps 50 --reps 2 2>&1 | grep -E "phase profile|advance" | tail -6
