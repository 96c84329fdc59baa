python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pd_build.log 2>&1 || exit 1
VXB_PROF_DUMP=gpurun_out/prof_c2.bin timeout 300 python tools/phase_profile.py --steps 100 --reps 1 2>&1 | tail -2
