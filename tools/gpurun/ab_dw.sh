for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_dw*.so; do
 echo "$f c3 $(VXB_LIB=$f timeout 900 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz 2>&1 | tail -1 | cut -c1-40) c2 $(VXB_LIB=$f timeout 600 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz 2>&1 | tail -1 | cut -c1-40)"
done
