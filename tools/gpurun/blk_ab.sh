# L2 block size for config 3 after the L2-policy changes (neurons per block).
for bn in 3000000 4000000 5000000 6700000; do
VXB_BLOCK_NEURONS=$bn timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/blk_$bn.log 2>&1; echo "c3 block=$bn $(tail -1 gpurun_out/blk_$bn.log | cut -c1-50)"; done
