# Bulk-copy ring depth / stage size A/B on config 2 and 3.
for rep in 1 2; do for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_s6.so build/variants/libvxb_s3.so build/variants/libvxb_e1024.so build/variants/libvxb_e512.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz > gpurun_out/st_$v.log 2>&1; echo "c2 $v $(tail -1 gpurun_out/st_$v.log | cut -c1-60)"; done; done
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_s6.so build/variants/libvxb_e1024.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/st3_$v.log 2>&1; echo "c3 $v $(tail -1 gpurun_out/st3_$v.log | cut -c1-60)"; done
