for fp in 0 1 2; do echo "== fpol $fp"; VXB_TUNING=1 VXB_FPOL=$fp timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance | tail -2; done
echo "== persist 0"; VXB_TUNING=1 VXB_PERSIST=0 timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance | tail -2
