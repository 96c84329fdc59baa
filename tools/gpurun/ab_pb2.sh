timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -1
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_head.so; do
 echo "$f c2 $(VXB_LIB=$f timeout 600 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz 2>&1 | tail -1 | cut -c1-45) c3 $(VXB_LIB=$f timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz 2>&1 | tail -1 | cut -c1-45)"
done
