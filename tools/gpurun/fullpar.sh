# full-size config 2 parity vs the reference (300 steps); only on a host with >= 150 GB
free -g | head -2; nproc
mem=$(free -g | awk '/^Mem:/{print $2}')
if [ "$mem" -lt 150 ]; then echo "host has ${mem} GB: skipped"; exit 0; fi
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fp_build.log 2>&1 || exit 1
timeout 3000 python -m pytest -q -p no:cacheprovider -rA tests/test_headline_parity_gpu.py -k full_size --durations=3 > gpurun_out/fp_test.log 2>&1; echo rc=$?; tail -8 gpurun_out/fp_test.log
