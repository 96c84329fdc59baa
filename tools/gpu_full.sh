# Full round-end style run: GPU tests (incl. multi-GPU), scaling bench, config3/4.
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/r_c2_n1.log 2>&1; echo c2n1=$?
for n in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n > gpurun_out/r_c2_n$n.log 2>&1; echo c2n$n=$?; done
timeout 900 python bench.py --workload config3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r_c3_n1.log 2>&1; echo c3n1=$?
for n in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr 127.0.0.1 --master-port 2972$n bench.py --gpus $n --workload config3 --steps 3 --warmup 3 > gpurun_out/r_c3_n$n.log 2>&1; echo c3n$n=$?; done
for r in 7 15 30; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 297$r bench.py --gpus 4 --workload config4 --rate $r --steps 3 --warmup 3 > gpurun_out/r_c4_r$r.log 2>&1; echo c4r$r=$?; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r_ref.log 2>&1; echo ref=$?
for f in r_c2_n1 r_c2_n2 r_c2_n4 r_c3_n1 r_c3_n2 r_c3_n4 r_c4_r7 r_c4_r15 r_c4_r30 r_ref; do tail -1 gpurun_out/$f.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$f', d['n_gpus'],'%.4g'%d['value'],'%.4f'%d.get('wall_s_per_bio_s',0),'%.2f'%d.get('exposed_exchange_us_per_step',0),'%.2f'%d.get('mean_rate_hz',0),'%.3f'%d.get('roofline',{}).get('frac',0), d.get('cpu_baseline',{}).get('value'))"; done
