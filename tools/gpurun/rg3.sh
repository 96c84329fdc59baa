echo "== base"; timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep -E "advance" | tail -2
for v in u5 u6 u8 l1pf; do echo "== $v"; VXB_LIB=build/variants/libvxb_$v.so timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance | tail -2; done
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_headline_parity_gpu.py tests/test_engine_gpu.py tests/test_timings_gpu.py 2>&1 | tail -2
