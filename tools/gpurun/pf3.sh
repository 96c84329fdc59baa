VXB_PROF_DUMP=gpurun_out/prof_c2.bin timeout 300 python tools/phase_profile.py --steps 100 --reps 2 2>&1 | tail -1; python tools/prof_analyze.py gpurun_out/prof_c2.bin 2>&1 | head -6
timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance
timeout 900 python -m pytest -x -q -p no:cacheprovider -m gpu tests 2>&1 | tail -2
