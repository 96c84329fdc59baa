timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for hv in 1 0; do
VXB_HELP=$hv VXB_PHASE_PROFILE=1 timeout 900 python tools/decompose.py config3 --steps 20 --reps 1 --only 10hz 2>&1 | grep -E "profile|10hz" | tail -2
VXB_HELP=$hv VXB_PHASE_PROFILE=1 timeout 900 python tools/decompose.py config2 --steps 100 --reps 1 --only 10hz 2>&1 | grep -E "profile|10hz" | tail -2
done
