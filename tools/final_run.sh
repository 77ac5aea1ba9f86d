set -x
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin/smi.txt
nproc >> gpurun_out/fin/smi.txt
python paper_2110_02140_b200/build.py > gpurun_out/fin/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/fin/ours_w1.json 2> gpurun_out/fin/ours_w1.err
timeout 400 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/fin/ref_w1.json 2> gpurun_out/fin/ref_w1.err
for N in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N > gpurun_out/fin/ours_w$N.json 2> gpurun_out/fin/ours_w$N.err
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $N --impl reference --steps 20 --warmup 3 > gpurun_out/fin/ref_w$N.json 2> gpurun_out/fin/ref_w$N.err
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 4 --config lstm_rows_zipf --no-cpu-baseline > gpurun_out/fin/lstm_rows_zipf_w4.json 2> gpurun_out/fin/lstm_rows_zipf_w4.err
timeout 300 python bench.py --config lstm_rows_zipf --no-cpu-baseline > gpurun_out/fin/lstm_rows_zipf_w1.json 2> gpurun_out/fin/lstm_rows_zipf_w1.err
tail -3 gpurun_out/fin/pytest_gpu.log
