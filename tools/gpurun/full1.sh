# full round check on one GPU: build, pytest -m gpu, smoke, bench line, ncu launch list + one full capture
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1 || { tail -20 gpurun_out/f_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rfE > gpurun_out/f_tests.log 2>&1; echo tests_rc=$?
tail -12 gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/f_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/f_bench.log | cut -c1-600
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/f_ncu_launch.log 2>&1; echo ncu_launch_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_kernel -s 3 -c 1 \
  -o gpurun_out/f_tile_full -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/f_ncu_full.log 2>&1; echo ncu_full_rc=$?
fi
