for lib in paper_2308_01241_b200/libvxb.so build/variants/libvxb_head.so; do echo "== $lib"
VXB_LIB=$lib timeout 600 python tools/phase_profile.py --workload config3 --steps 20 --reps 2 2>&1 | grep -E "advance" | tail -1
VXB_LIB=$lib timeout 600 python tools/phase_profile.py --workload config3 --steps 20 --reps 2 --silent 2>&1 | grep -E "advance" | tail -1
VXB_LIB=$lib VXB_TUNING=1 VXB_PATH=l2 timeout 600 python tools/phase_profile.py --steps 50 --reps 2 2>&1 | grep -E "advance" | tail -1
done
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_headline_parity_gpu.py tests/test_engine_gpu.py 2>&1 | tail -2
timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep -E "advance" | tail -2
