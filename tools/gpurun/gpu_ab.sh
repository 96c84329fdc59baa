# A/B the kernel variants in build/variants on config 2 (after a parity pass)
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "not acceptance" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_*.so; do v=$(basename $f .so); VXB_LIB=$f timeout 300 python tools/decompose.py > gpurun_out/ab_$v.log 2>&1; echo "$v rc=$? $(cat gpurun_out/ab_$v.log | tail -1)"; done
