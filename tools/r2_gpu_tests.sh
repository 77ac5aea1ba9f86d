# round-2 GPU check: full -m gpu suite (1 GPU) + smoke
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r2_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2_pytest.log
