# Occupancy variants: config 3 (update-heavy, 1 GPU) and config 2.
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_m4.so build/variants/libvxb_t384m2.so build/variants/libvxb_t320m3.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 > gpurun_out/occ3_$v.log 2>&1; echo "c3 $v $(tail -1 gpurun_out/occ3_$v.log | cut -c1-200)"
VXB_LIB=$f timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 > gpurun_out/occ2_$v.log 2>&1; echo "c2 $v $(tail -1 gpurun_out/occ2_$v.log | cut -c1-200)"
done
