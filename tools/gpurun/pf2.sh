VXB_PROF_DUMP=gpurun_out/prof_c2.bin timeout 300 python tools/phase_profile.py --steps 100 --reps 2 2>&1 | tail -1; python tools/prof_analyze.py gpurun_out/prof_c2.bin 2>&1 | head -4
for v in nofuse; do echo "== $v"; VXB_LIB=build/variants/libvxb_$v.so timeout 300 python tools/phase_profile.py --steps 100 --reps 2 2>&1 | tail -1; done
timeout 600 python -m pytest -x -q -p no:cacheprovider tests/test_headline_parity_gpu.py tests/test_engine_gpu.py 2>&1 | tail -2
