# Half of config 5 on 4 GPUs: block count per rank (default ceil(n / 4.19M): 6/6/6/7) vs forced equal blocks.
for bn in 0 5100000 3600000; do
if [ $bn = 0 ]; then unset VXB_BLOCK_NEURONS; else export VXB_BLOCK_NEURONS=$bn; fi
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29860 + bn % 7)) bench.py --gpus 4 --workload config4 --rate 15 --neurons 100000000 --steps 2 --warmup 3 --bio-ms 50 --no-cpu > gpurun_out/c5b_$bn.log 2>&1
echo "block=$bn $(grep -h '"metric"' gpurun_out/c5b_$bn.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.4g'%d['value'], d['wall_s_per_bio_s'], d['exposed_exchange_us_per_step'])")"
done
