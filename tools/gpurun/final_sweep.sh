# Round-end evidence on a 4-GPU box: GPU tests (incl. multi-GPU), smoke, the
# default bench, config 2 weak scaling, config 3 strong scaling, config 4 rate
# sweep, the reference arm, then the ncu launch list + one full capture.
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/fs_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/fs_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fs_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/fs_smoke.log
python bench.py > gpurun_out/fs_c2_n1.log 2>&1; echo c2n1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 --no-cpu > gpurun_out/fs_c2_n2.log 2>&1; echo c2n2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29814 bench.py --gpus 4 --no-cpu > gpurun_out/fs_c2_n4.log 2>&1; echo c2n4=$?
timeout 900 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu > gpurun_out/fs_c3_n1.log 2>&1; echo c3n1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29822 bench.py --gpus 2 --workload config3 --steps 3 --warmup 3 > gpurun_out/fs_c3_n2.log 2>&1; echo c3n2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29824 bench.py --gpus 4 --workload config3 --steps 3 --warmup 3 > gpurun_out/fs_c3_n4.log 2>&1; echo c3n4=$?
for r in 7 15 30; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 2983$((r % 10)) bench.py --gpus 4 --workload config4 --rate $r --steps 3 --warmup 3 > gpurun_out/fs_c4_r$r.log 2>&1; echo c4r$r=$?; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fs_ref.log 2>&1; echo ref=$?
for f in fs_c2_n1 fs_c2_n2 fs_c2_n4 fs_c3_n1 fs_c3_n2 fs_c3_n4 fs_c4_r7 fs_c4_r15 fs_c4_r30 fs_ref; do tail -1 gpurun_out/$f.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$f', d['n_gpus'],'%.4g'%d['value'],'%.4f'%d.get('wall_s_per_bio_s',0),'%.2f'%d.get('exposed_exchange_us_per_step',0),'%.2f'%d.get('mean_rate_hz',0),'%.3f'%d.get('roofline',{}).get('frac',0), d.get('e2e',{}).get('value'), d.get('cpu_baseline',{}).get('value'))" 2>&1 | tail -1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fs_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/fs_ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/fs_step python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/fs_ncu_full.log 2>&1; echo ncu_full=$?
