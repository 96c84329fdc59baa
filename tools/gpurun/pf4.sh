echo "== silent"; VXB_PROF_DUMP=gpurun_out/prof_silent.bin timeout 300 python tools/phase_profile.py --steps 100 --reps 2 --silent 2>&1 | grep advance | tail -1; python tools/prof_analyze.py gpurun_out/prof_silent.bin 2>&1 | sed -n 2,3p
for v in u8; do echo "== $v"; VXB_LIB=build/variants/libvxb_$v.so timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance; done
echo "== base"; timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance
