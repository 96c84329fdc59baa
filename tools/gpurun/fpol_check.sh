# Automatic evict_last update stream: parity subset, config 2 decompose, default bench, 2-GPU config 2.
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "not noise" > gpurun_out/pytest_fpol.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_fpol.log
VXB_VERBOSE=1 timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz 2>&1 | tail -1 | cut -c1-80
python bench.py --no-cpu > gpurun_out/fpol_bench.log 2>&1; grep -h '"metric"' gpurun_out/fpol_bench.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench', '%.4g'%d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 2 --no-cpu --steps 10 > gpurun_out/fpol_mg.log 2>&1
grep -h '"metric"' gpurun_out/fpol_mg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2x2', '%.4g'%d['value'])"
