VXB_PROF_DUMP=gpurun_out/prof_c2.bin timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep -E "advance|phase profile" | tail -4; python tools/prof_analyze.py gpurun_out/prof_c2.bin 2>&1 | grep -v Warn | sed -n 2,3p
timeout 300 python tools/phase_profile.py --steps 100 --reps 2 --silent 2>&1 | grep -E "advance" | tail -1
timeout 900 python -m pytest -x -q -p no:cacheprovider -m gpu tests 2>&1 | tail -2
