# Delivery chunk cap: parity subset + config 2/3 step times, then 2-GPU config 2.
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "not noise" > gpurun_out/pytest_ch.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_ch.log
VXB_PHASE_PROFILE=1 timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz 2>&1 | grep -E "profile|10hz" | tail -2
timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz 2>&1 | tail -1
