# Synapse-stream policy (pol_syn) check: parity subset, config 2/3 A/B vs evict_first, 2-GPU config 2.
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "not noise" > gpurun_out/pytest_pol.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_pol.log
for rep in 1 2; do for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_polsf.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 300 python tools/decompose.py config2 --steps 100 --reps 3 --only 10hz > gpurun_out/pol_$v.log 2>&1; echo "c2 $v $(tail -1 gpurun_out/pol_$v.log | cut -c1-50)"; done; done
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_polsf.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 600 python tools/decompose.py config3 --steps 20 --reps 2 --only 10hz > gpurun_out/pol3_$v.log 2>&1; echo "c3 $v $(tail -1 gpurun_out/pol3_$v.log | cut -c1-50)"; done
for rep in 1 2; do for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_polsf.so; do v=$(basename $f .so)
VXB_LIB=$f timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port $((29600 + rep)) bench.py --gpus 2 --no-cpu --steps 10 > gpurun_out/polmg_$v.log 2>&1
echo "c2x2 $v $(grep -h '"metric"' gpurun_out/polmg_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('%.4g'%d['value'])")"; done; done
