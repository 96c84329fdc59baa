timeout 600 python tools/phase_profile.py --workload config3 --steps 20 --reps 2 2>&1 | grep -E "advance" | tail -1
timeout 600 python tools/phase_profile.py --workload config3 --steps 20 --reps 2 --silent 2>&1 | grep -E "advance" | tail -1
timeout 900 python -m pytest -x -q -p no:cacheprovider -m gpu tests 2>&1 | tail -2
