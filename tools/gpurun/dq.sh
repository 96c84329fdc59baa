timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance | tail -2
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_headline_parity_gpu.py tests/test_engine_gpu.py 2>&1 | tail -2
