# tile_mp vs l2 on config-2-shaped shards of 2M and 4M neurons
for v in 200 400; do
  echo "== voxels $v"
  timeout 600 python tools/phase_profile.py --voxels $v --steps 20 --reps 2 2>&1 | grep -E "phase profile|advance|kernel" | tail -3
  timeout 600 python tools/phase_profile.py --voxels $v --steps 20 --reps 2 --path l2 2>&1 | grep -E "phase profile|advance" | tail -2
done
