VXB_PROF_DUMP=gpurun_out/prof_c2.bin timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep -E "advance" | tail -2; python tools/prof_analyze.py gpurun_out/prof_c2.bin 2>&1 | grep -v Warn | sed -n 2,3p
echo "== nostream1"; VXB_LIB=build/variants/libvxb_nostream1.so timeout 300 python tools/phase_profile.py --steps 100 --reps 3 2>&1 | grep advance | tail -2
timeout 900 python -m pytest -x -q -p no:cacheprovider tests/test_headline_parity_gpu.py tests/test_engine_gpu.py tests/test_timings_gpu.py 2>&1 | tail -2
