timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
timeout 900 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz 2>&1 | tail -1
timeout 600 python tools/decompose.py config2 --steps 100 --reps 3 2>&1 | tail -1
