for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_head.so; do
 VXB_VERBOSE=1 VXB_LIB=$f timeout 600 python tools/decompose.py config2 --steps 100 --reps 2 --only 10hz 2>&1 | tail -2 | cut -c1-200
done
