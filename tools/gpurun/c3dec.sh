timeout 900 python tools/decompose.py config3 --steps 20 --reps 2 > gpurun_out/c3_dec.log 2>&1; echo dec=$?; tail -1 gpurun_out/c3_dec.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -c 1 -o gpurun_out/c3_step python tools/decompose.py config3 --steps 10 --reps 1 --only 10hz > gpurun_out/c3_ncu.log 2>&1; echo ncu=$?; tail -2 gpurun_out/c3_ncu.log
