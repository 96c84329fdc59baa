# ncu --set full of the barrier-free tile kernel (config 2, one 20-step launch)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu_build.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_kernel -c 1 \
  -o gpurun_out/tile_nb -f python tools/phase_profile.py --steps 20 --reps 1 > gpurun_out/ncu_nb.log 2>&1
echo ncu_rc=$?; tail -3 gpurun_out/ncu_nb.log
