# L2 block size 64 vs 80 MB with equal block counts across ranks: config 3 (1/2/4 GPUs), half of config 5 (4 GPUs).
for mb in 64 80; do export VXB_BLOCK_MB=$mb
timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/bm3_$mb.log 2>&1; echo "c3 n1 mb=$mb $(tail -1 gpurun_out/bm3_$mb.log | cut -c1-50)"
for g in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$g --master-addr 127.0.0.1 --master-port $((29870 + g + mb)) bench.py --gpus $g --workload config3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bm3_${mb}_$g.log 2>&1
echo "c3 n$g mb=$mb $(grep -h '"metric"' gpurun_out/bm3_${mb}_$g.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.4g'%d['value'], d['wall_s_per_bio_s'], d['exposed_exchange_us_per_step'])")"; done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port $((29890 + mb)) bench.py --gpus 4 --workload config4 --rate 15 --neurons 100000000 --steps 2 --warmup 3 --bio-ms 50 --no-cpu > gpurun_out/bm5_$mb.log 2>&1
echo "c5half mb=$mb $(grep -h '"metric"' gpurun_out/bm5_$mb.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.4g'%d['value'], d['wall_s_per_bio_s'], d['exposed_exchange_us_per_step'])")"
done
