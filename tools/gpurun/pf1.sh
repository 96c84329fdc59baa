for c in 12 8 16; do echo "== cons $c"; VXB_PROF_DUMP=gpurun_out/prof_c2_$c.bin timeout 300 python tools/phase_profile.py --steps 100 --reps 1 --cons $c 2>&1 | tail -1; python tools/prof_analyze.py gpurun_out/prof_c2_$c.bin | head -3; done
for v in nopf bw4; do echo "== $v"; VXB_LIB=build/variants/libvxb_$v.so timeout 300 python tools/phase_profile.py --steps 100 --reps 1 2>&1 | tail -1; done
