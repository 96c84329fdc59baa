# Dynamic vs static delivery deal on L2-blocked multi-GPU runs (config 3 at 2/4 GPUs, half of config 5).
for d in 0 1; do export VXB_DYN=$d
for g in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$g --master-addr 127.0.0.1 --master-port $((29920 + g + 10 * d)) bench.py --gpus $g --workload config3 --steps 3 --warmup 3 --no-cpu > gpurun_out/dyn3_${d}_$g.log 2>&1
echo "c3 n$g dyn=$d $(grep -h '"metric"' gpurun_out/dyn3_${d}_$g.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.4g'%d['value'], d['wall_s_per_bio_s'], d['exposed_exchange_us_per_step'])")"; done
done
