for b in 3145728 2097152 1572864 1048576 786432; do
 echo "block $b $(VXB_BLOCK_NEURONS=$b timeout 900 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz 2>&1 | tail -1)"
done
