# config 5 shape on one GPU (25M neurons, 1000-voxel DTI-like, K=500, 15 Hz) and silent
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5_build.log 2>&1 || { tail -20 gpurun_out/c5_build.log; exit 1; }
summ() { grep '^{' $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','ms_per_step','wall_s_per_bio_s','mean_rate_hz','device_memory_used_gb']}, d['config']['schedule'])"; }
timeout 1800 python bench.py --workload config5 --steps 5 --warmup 3 --no-cpu > gpurun_out/c5_one.log 2>&1; echo rc=$?; summ gpurun_out/c5_one.log
timeout 1800 python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu > gpurun_out/c3_one.log 2>&1; echo rc=$?; summ gpurun_out/c3_one.log
