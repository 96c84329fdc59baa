# ncu --set full of one config-3 step_kernel launch, silent network (update only) and 10 Hz.
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o gpurun_out/c3_silent python tools/decompose.py config3 --steps 5 --reps 1 --only silent > gpurun_out/c3s_ncu.log 2>&1; echo ncu_silent=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o gpurun_out/c3_10hz python tools/decompose.py config3 --steps 5 --reps 1 --only 10hz > gpurun_out/c3h_ncu.log 2>&1; echo ncu_10hz=$?
