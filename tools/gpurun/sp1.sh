echo "== base"; timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep -E "advance" | tail -2
for v in spin2 spin3; do echo "== $v"; VXB_LIB=build/variants/libvxb_$v.so timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance | tail -2; done
echo "== base"; timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep -E "advance" | tail -2
