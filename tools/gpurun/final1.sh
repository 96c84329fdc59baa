# final 1-GPU evidence at HEAD: GPU tests, smoke, bench (config 2), launch list, ncu of the tile kernel
ts() { date +%T; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f1_build.log 2>&1 || { tail -20 gpurun_out/f1_build.log; exit 1; }
echo "$(ts) tests"; timeout 1500 python -m pytest -q -p no:cacheprovider -m gpu tests > gpurun_out/f1_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/f1_tests.log
echo "$(ts) smoke"; timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/f1_smoke.log
echo "$(ts) bench"; timeout 900 python bench.py > gpurun_out/f1_bench.log 2>&1; echo bench_rc=$?; grep '^{' gpurun_out/f1_bench.log | tail -1 | cut -c1-200
echo "$(ts) bench ref"; timeout 900 python bench.py --impl reference > gpurun_out/f1_bench_ref.log 2>&1; echo ref_rc=$?; grep '^{' gpurun_out/f1_bench_ref.log | tail -1 | cut -c1-200
echo "$(ts) launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/f1_launch_run.log 2>&1; echo rc=$?
echo "$(ts) ncu"; timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_kernel -s 3 -c 1 -o gpurun_out/f1_tile -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/f1_ncu.log 2>&1; echo rc=$?
echo "$(ts) done"
