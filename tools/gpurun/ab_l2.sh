for cfg in "VXB_PERSIST=1 VXB_FPOL=0" "VXB_PERSIST=1 VXB_FPOL=1"; do
  c3=$(env $cfg timeout 600 python bench.py --workload config3 --steps 2 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print("c3 %.3f s/bio-s"%d["wall_s_per_bio_s"])')
  echo "$cfg $c3"
done
