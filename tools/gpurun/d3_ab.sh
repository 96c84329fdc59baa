# Update load pipeline depth: default (one chunk ahead, 3 CTAs/SM) vs two chunks ahead (d3: spills at the 80-register cap;
# d3m2: 2 CTAs/SM, no cap) vs 2 CTAs/SM alone (m2); config 3 (silent + 10 Hz) and config 2. Parity of d3 and d3m2 first.
for v in d3 d3m2; do VXB_LIB=build/variants/libvxb_$v.so timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_$v.log 2>&1; echo "pytest $v=$? $(tail -1 gpurun_out/pytest_$v.log)"; done
for rep in 1 2; do for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_d3.so build/variants/libvxb_d3m2.so build/variants/libvxb_m2.so; do v=$(basename $f .so)
 echo "$v c3 $(VXB_LIB=$f timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 2>&1 | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print({k:round(x["us_per_step"],1) for k,x in d.items()})')"
 echo "$v c2 $(VXB_LIB=$f timeout 600 python tools/decompose.py config2 --steps 100 --reps 3 2>&1 | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print({k:round(x["us_per_step"],1) for k,x in d.items()})')"
done; done
