# final multi-GPU evidence: tests on 4 GPUs, config 2 at 2 GPUs, config 2 / 3 / 5 at 4 GPUs
ts() { date +%T; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f4_build.log 2>&1 || { tail -20 gpurun_out/f4_build.log; exit 1; }
echo "$(ts) tests"; timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE > gpurun_out/f4_tests.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/f4_tests.log
echo "$(ts) c2 n2"; timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/f2_c2.log 2>&1; echo rc=$?; grep '^{' gpurun_out/f2_c2.log | tail -1 | cut -c1-120
for w in config2 config3 config5; do
  echo "$(ts) $w"; timeout 2400 python bench.py --gpus 4 --workload $w --steps 10 --warmup 3 --no-cpu > gpurun_out/f4_$w.log 2>&1; echo "$w rc=$?"; grep '^{' gpurun_out/f4_$w.log | tail -1 | cut -c1-120
done
echo "$(ts) done"
