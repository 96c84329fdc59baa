# tile-path phase profile (config 2): consumer-warp sweep, silent run, l2 path
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1 || { tail -20 gpurun_out/p_build.log; exit 1; }
for c in 8 12 16 20; do echo "== cons $c"; timeout 600 python tools/phase_profile.py --steps 50 --reps 2 --cons $c 2>&1 | tail -4; done
timeout 600 python tools/phase_profile.py --steps 50 --silent --reps 1 2>&1 | tail -2
