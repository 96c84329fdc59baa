# pytest -m gpu (all, no -x) + smoke on one GPU; logs under gpurun_out/
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider -rfE ${PYTEST_ARGS:-} > gpurun_out/t_tests.log 2>&1; echo tests_rc=$?
tail -15 gpurun_out/t_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t_smoke.log 2>&1; echo smoke_rc=$?
