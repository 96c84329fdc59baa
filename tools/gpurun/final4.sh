# final 4-GPU evidence: multi-GPU tests, bench lines config 2 / 3 / 5 (4 GPUs)
ts() { date +%T; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f4_build.log 2>&1 || { tail -20 gpurun_out/f4_build.log; exit 1; }
echo "$(ts) tests"; timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rfE > gpurun_out/f4_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/f4_tests.log
for w in config2 config3 config5; do
  echo "$(ts) $w"; timeout 2400 python bench.py --gpus 4 --workload $w --steps ${STEPS:-10} --warmup 3 --no-cpu > gpurun_out/f4_$w.log 2>&1; echo "$w rc=$?"; grep '^{' gpurun_out/f4_$w.log | tail -1 | cut -c1-160
done
echo "$(ts) done"
