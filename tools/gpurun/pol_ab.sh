# L2 policy of the synapse stream: evict_first (default) vs evict_normal, +/- evict_first update stream.
for rep in 1 2 3; do
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_polsn.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz > gpurun_out/pol_$v.log 2>&1; echo "c2 $v $(tail -1 gpurun_out/pol_$v.log | cut -c1-50)"
VXB_FPOL=1 VXB_LIB=$f timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz > gpurun_out/polf_$v.log 2>&1; echo "c2 fpol $v $(tail -1 gpurun_out/polf_$v.log | cut -c1-50)"
done; done
