VXB_PROF_DUMP=gpurun_out/prof4.bin timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29561 tools/phase_profile.py --steps 100 --reps 2 2>&1 | grep -E "advance|phase profile" | tail -6
for r in 0 1 2 3; do echo "== rank $r"; python tools/prof_analyze.py gpurun_out/prof4.bin.rank$r 2>&1 | grep -v Warn | sed -n 2,6p; done
