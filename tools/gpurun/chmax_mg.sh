# Local-list chunk cap on 2 GPUs (config 2 weak): CH <= 1 vs <= 32, alternating.
for rep in 1 2 3; do for c in 1 32; do
VXB_CHMAX=$c timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29700 + c + 100 * rep)) bench.py --gpus 2 --no-cpu --steps 10 > gpurun_out/chm_$c.log 2>&1
echo "ch$c $(grep -h '"metric"' gpurun_out/chm_$c.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.4g'%d['value'], d['exposed_exchange_us_per_step'])")"
done; done
