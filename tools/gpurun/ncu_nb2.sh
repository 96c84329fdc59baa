# ncu --set full of the tile kernel (config 2, one 20-step launch) + launch list of the bench
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_kernel -c 1 \
  -o gpurun_out/tile_r02b -f python tools/phase_profile.py --steps 20 --reps 1 > gpurun_out/ncu_nb2.log 2>&1
echo ncu_rc=$?; tail -2 gpurun_out/ncu_nb2.log
