for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_xifast.so paper_2308_01241_b200/libvxb.so build/variants/libvxb_xifast.so; do
 echo "$f $(VXB_LIB=$f timeout 600 python bench.py --no-cpu 2>&1 | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print("%.4g"%d["value"], d["ms_per_step"])') $(VXB_LIB=$f timeout 600 python tools/decompose.py config3 --steps 20 --reps 1 --only silent 2>&1 | tail -1 | cut -c1-50)"
done
