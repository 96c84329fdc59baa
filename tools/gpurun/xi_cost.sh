# Cost of the OU noise in the update (diagnostic variants, not parity-preserving): default vs fp64 Box-Muller without
# the correct-rounding check (xifast) vs no noise (xizero); config 2 (10 Hz + silent) and config 3 (10 Hz + silent).
for rep in 1 2; do for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_xifast.so build/variants/libvxb_xizero.so; do
 echo "$(basename $f) c2 $(VXB_LIB=$f timeout 600 python tools/decompose.py config2 --steps 100 --reps 3 2>&1 | tail -1 | cut -c1-160)"
 echo "$(basename $f) c3 $(VXB_LIB=$f timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 2>&1 | tail -1 | cut -c1-160)"
done; done
