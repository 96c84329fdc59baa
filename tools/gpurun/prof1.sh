# tile-path phase profile (config 2): consumer-warp sweep, silent run, then a few parity tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1 || { tail -20 gpurun_out/p_build.log; exit 1; }
for c in ${CONS:-6 9 12 16}; do echo "== cons $c"; timeout 600 python tools/phase_profile.py --steps 50 --reps 2 --cons $c 2>&1 | tail -4; done
timeout 600 python tools/phase_profile.py --steps 50 --silent --reps 1 2>&1 | tail -2
timeout 900 python -m pytest -x -q -p no:cacheprovider -rfE \
  "tests/test_engine_gpu.py::test_matches_reference_bit_for_bit_six_neurons" \
  "tests/test_engine_gpu.py::test_ring_multiworker_both_paths" \
  "tests/test_engine_gpu.py::test_advance_without_forced_spikes_or_injection_after_one_with" \
  "tests/test_headline_parity_gpu.py::test_config2_regime_ring12_k1000_one_bio_second" 2>&1 | tail -5
