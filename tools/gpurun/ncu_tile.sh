# one ncu --set full capture of the tile kernel (config 2, 20-step advance)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1 || { tail -20 gpurun_out/n_build.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_kernel -s 1 -c 1 \
  -o gpurun_out/tile_full -f python tools/phase_profile.py --steps 20 --reps 2 > gpurun_out/n_ncu.log 2>&1; echo ncu_rc=$?
tail -5 gpurun_out/n_ncu.log
