for b in 5000000 6666667 10000000 20000000; do
 echo "block $b $(VXB_BLOCK_NEURONS=$b VXB_PHASE_PROFILE=1 timeout 900 python tools/decompose.py config3 --steps 20 --reps 1 --only 10hz 2>&1 | grep -E 'profile|10hz' | tail -2 | cut -c1-130 | tr '\n' ' ')"
done
