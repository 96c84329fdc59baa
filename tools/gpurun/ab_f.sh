timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/decompose.py config3 --steps 20 --reps 2 2>&1 | tail -1
timeout 600 python tools/decompose.py config2 --steps 100 --reps 3 2>&1 | tail -1
timeout 600 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2', '%.4g'%d['value'], d['ms_per_step'])"
timeout 900 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3', '%.4g'%d['value'], d['wall_s_per_bio_s'])"
