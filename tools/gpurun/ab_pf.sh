timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_nopf.so; do
 echo $f
 VXB_LIB=$f timeout 900 python tools/decompose.py config3 --steps 20 --reps 2 2>&1 | tail -1
 VXB_LIB=$f timeout 600 python tools/decompose.py config2 --steps 100 --reps 3 2>&1 | tail -1
done
