# A/B kernel variants on config 3 (20M neurons, 1 GPU) and config 2
for f in paper_2308_01241_b200/libvxb.so build/variants/libvxb_*.so; do v=$(basename $f .so)
  VXB_LIB=$f timeout 600 python bench.py --workload config3 --steps 2 --warmup 3 --no-cpu > gpurun_out/ab3_$v.log 2>&1
  VXB_LIB=$f timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ab2_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/ab3_$v.log | python -c 'import json,sys;d=json.loads(sys.stdin.read());print("c3 %.3f s/bio-s"%d["wall_s_per_bio_s"])') $(tail -1 gpurun_out/ab2_$v.log | python -c 'import json,sys;d=json.loads(sys.stdin.read());print("c2 %.4g ev/s %.1f us/step"%(d["value"],d["ms_per_step"]*10))')"
done
