VXB_VERBOSE=1 timeout 900 python tools/decompose.py config3 --steps 20 --reps 1 --only silent 2>&1 | tail -3
VXB_VERBOSE=1 timeout 900 python tools/decompose.py config2 --steps 20 --reps 1 --only silent 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o gpurun_out/c3_silent3 python tools/decompose.py config3 --steps 5 --reps 1 --only silent > gpurun_out/c3s_ncu.log 2>&1; echo ncu=$?
