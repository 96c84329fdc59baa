timeout 600 python -m pytest tests/test_engine_gpu.py -x -q 2>&1 | tail -2
timeout 900 python tools/decompose.py config3 --steps 20 --reps 2 2>&1 | tail -1
for d in 0 1; do VXB_DYN=$d timeout 600 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2 dyn=$d', '%.4g'%d['value'], d['ms_per_step'])"; done
timeout 900 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3', '%.4g'%d['value'], d['wall_s_per_bio_s'])"
