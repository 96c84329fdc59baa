for d in 0 1; do
 VXB_PHASE_PROFILE=1 VXB_DYN=$d timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29771 bench.py --gpus 4 --workload config3 --steps 2 --warmup 3 > gpurun_out/mg_c3_n4_p$d.log 2>&1; echo "dyn=$d rc=$?"; grep "phase profile" gpurun_out/mg_c3_n4_p$d.log | tail -8
done
