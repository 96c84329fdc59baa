VXB_PROF_DUMP=gpurun_out/prof_c2.bin timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep -E "advance|phase profile" | tail -3; python tools/prof_analyze.py gpurun_out/prof_c2.bin 2>&1 | head -6
timeout 900 python -m pytest -x -q -p no:cacheprovider -m gpu tests 2>&1 | tail -2
