set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest1.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/r2_pytest1.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo bench_rc=$?
cat gpurun_out/r2_bench1.json
