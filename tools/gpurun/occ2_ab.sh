# Occupancy variants after the L2-policy changes (config 2, config 3).
for rep in 1 2; do for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_t384m2.so build/variants/libvxb_t320m3.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz > gpurun_out/o2_$v.log 2>&1; echo "c2 $v $(tail -1 gpurun_out/o2_$v.log | cut -c1-50)"; done; done
