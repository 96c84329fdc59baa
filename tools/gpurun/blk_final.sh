# Block-size rule check: parity (full-size + multi-GPU), half of config 5 and config 3 at 4 GPUs with the defaults.
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_multigpu.py -q -p no:cacheprovider > gpurun_out/pytest_blk.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_blk.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 4 --workload config4 --rate 15 --neurons 100000000 --steps 2 --warmup 3 --bio-ms 50 > gpurun_out/c5_half.log 2>&1
echo "c5half $(grep -h '"metric"' gpurun_out/c5_half.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.4g'%d['value'], d['wall_s_per_bio_s'], d['exposed_exchange_us_per_step'])")"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29912 bench.py --gpus 4 --workload config3 --steps 3 --warmup 3 --no-cpu > gpurun_out/c3_n4.log 2>&1
echo "c3n4 $(grep -h '"metric"' gpurun_out/c3_n4.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.4g'%d['value'], d['wall_s_per_bio_s'], d['exposed_exchange_us_per_step'])")"
