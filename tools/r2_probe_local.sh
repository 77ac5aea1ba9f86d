python paper_2110_02140_b200/build.py > /dev/null 2>&1
python tools/local_probe.py
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_full.log
tail -n 4 gpurun_out/r2_pytest_full.log
