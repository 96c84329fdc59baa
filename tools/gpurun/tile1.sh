# quick tile-path check: build, a few parity tests, then the bench line
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1 || { tail -20 gpurun_out/k_build.log; exit 1; }
timeout 900 python -m pytest -x -q -p no:cacheprovider -rfE \
  "tests/test_engine_gpu.py::test_matches_reference_bit_for_bit_six_neurons" \
  "tests/test_engine_gpu.py::test_ring_multiworker_both_paths" \
  "tests/test_engine_gpu.py::test_config1_one_bio_second" \
  tests/test_headline_parity_gpu.py > gpurun_out/k_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/k_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/k_bench.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/k_bench.log | cut -c1-1500
