# Half of config 5 on 4 GPUs: 100M neurons x K=500 = 5e10 synapses, 15 Hz point
VXB_VERBOSE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29851 bench.py --gpus 4 --workload config4 --rate 15 --neurons 100000000 --steps 2 --warmup 3 --bio-ms 50 > gpurun_out/c5_half.log 2>&1; echo rc=$?
grep "vxb:" gpurun_out/c5_half.log | head -4
tail -1 gpurun_out/c5_half.log | cut -c1-600
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
