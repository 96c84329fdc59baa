# Knobs after the L2-policy changes: persisting carve-out off, delivery warps 4 / 2; config 2 and 3.
for rep in 1 2; do
VXB_PERSIST=0 timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz > gpurun_out/kn_p0.log 2>&1; echo "c2 persist0 $(tail -1 gpurun_out/kn_p0.log | cut -c1-60)"
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_dw4.so build/variants/libvxb_dw2.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz > gpurun_out/kn_$v.log 2>&1; echo "c2 $v $(tail -1 gpurun_out/kn_$v.log | cut -c1-60)"; done; done
VXB_PERSIST=0 timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/kn3_p0.log 2>&1; echo "c3 persist0 $(tail -1 gpurun_out/kn3_p0.log | cut -c1-60)"
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_dw4.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/kn3_$v.log 2>&1; echo "c3 $v $(tail -1 gpurun_out/kn3_$v.log | cut -c1-60)"; done
