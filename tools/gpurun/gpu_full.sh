# Round-end style run: GPU tests (incl. multi-GPU), scaling bench, config 3/4.
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/r_c2_n1.log 2>&1; echo c2n1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 > gpurun_out/r_c2_n2.log 2>&1; echo c2n2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29814 bench.py --gpus 4 > gpurun_out/r_c2_n4.log 2>&1; echo c2n4=$?
timeout 900 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r_c3_n1.log 2>&1; echo c3n1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29822 bench.py --gpus 2 --workload config3 --steps 3 --warmup 3 > gpurun_out/r_c3_n2.log 2>&1; echo c3n2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29824 bench.py --gpus 4 --workload config3 --steps 3 --warmup 3 > gpurun_out/r_c3_n4.log 2>&1; echo c3n4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29831 bench.py --gpus 4 --workload config4 --rate 7 --steps 3 --warmup 3 > gpurun_out/r_c4_r7.log 2>&1; echo c4r7=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29832 bench.py --gpus 4 --workload config4 --rate 15 --steps 3 --warmup 3 > gpurun_out/r_c4_r15.log 2>&1; echo c4r15=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29833 bench.py --gpus 4 --workload config4 --rate 30 --steps 3 --warmup 3 > gpurun_out/r_c4_r30.log 2>&1; echo c4r30=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r_ref.log 2>&1; echo ref=$?
for f in r_c2_n1 r_c2_n2 r_c2_n4 r_c3_n1 r_c3_n2 r_c3_n4 r_c4_r7 r_c4_r15 r_c4_r30 r_ref; do tail -1 gpurun_out/$f.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$f', d['n_gpus'],'%.4g'%d['value'],'%.4f'%d.get('wall_s_per_bio_s',0),'%.2f'%d.get('exposed_exchange_us_per_step',0),'%.2f'%d.get('mean_rate_hz',0),'%.3f'%d.get('roofline',{}).get('frac',0), d.get('e2e',{}).get('value'), d.get('cpu_baseline',{}).get('value'))"; done
# ncu: launch list of the default bench + one full capture of the step kernel
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/c2_step python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
