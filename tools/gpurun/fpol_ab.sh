# Update-stream L2 policy: evict_normal (0) vs evict_last (2) on config 2 (state fits L2) and config 3.
for rep in 1 2; do for fp in 0 2; do
VXB_FPOL=$fp timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 > gpurun_out/fpol_$fp.log 2>&1; echo "c2 fpol=$fp $(tail -1 gpurun_out/fpol_$fp.log | cut -c1-160)"; done; done
for fp in 0 2; do VXB_FPOL=$fp timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/fpol3_$fp.log 2>&1; echo "c3 fpol=$fp $(tail -1 gpurun_out/fpol3_$fp.log | cut -c1-60)"; done
