# round-2 evidence at HEAD (1 GPU): bench lines, launch list, ncu --set full of the
# dominant kernel per workload (config 2 tile_kernel, config 3 / 5 step_kernel)
set -u
ts() { date +%T; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev_build.log 2>&1 || { tail -20 gpurun_out/ev_build.log; exit 1; }
echo "$(ts) bench config2"; timeout 900 python bench.py > gpurun_out/ev_bench_c2.log 2>&1; echo rc=$?; grep '^{' gpurun_out/ev_bench_c2.log | tail -1 | cut -c1-300
echo "$(ts) launches"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ev_launch_run.log 2>&1; echo rc=$?
echo "$(ts) ncu c2"; timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_kernel -s 3 -c 1 -o gpurun_out/ev_c2_tile -f python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ev_ncu_c2.log 2>&1; echo rc=$?
echo "$(ts) bench config3"; timeout 1200 python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu > gpurun_out/ev_bench_c3.log 2>&1; echo rc=$?; grep '^{' gpurun_out/ev_bench_c3.log | tail -1 | cut -c1-300
echo "$(ts) ncu c3"; timeout 1200 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/ev_c3_step -f python bench.py --workload config3 --steps 1 --warmup 3 --no-cpu > gpurun_out/ev_ncu_c3.log 2>&1; echo rc=$?
echo "$(ts) bench config5"; timeout 1800 python bench.py --workload config5 --steps 3 --warmup 3 --no-cpu > gpurun_out/ev_bench_c5.log 2>&1; echo rc=$?; grep '^{' gpurun_out/ev_bench_c5.log | tail -1 | cut -c1-300
echo "$(ts) ncu c5"; timeout 1800 ncu --set full --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/ev_c5_step -f python bench.py --workload config5 --steps 1 --warmup 3 --no-cpu > gpurun_out/ev_ncu_c5.log 2>&1; echo rc=$?
echo "$(ts) done"
