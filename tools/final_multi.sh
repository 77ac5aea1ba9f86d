mkdir -p gpurun_out/fin
for N in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N > gpurun_out/fin/ours_w$N.json 2> gpurun_out/fin/ours_w$N.err
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 4 --config lstm_rows_zipf --no-cpu-baseline > gpurun_out/fin/lstm_rows_zipf_w4.json 2> gpurun_out/fin/lstm_rows_zipf_w4.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29536 bench.py --gpus 4 --config lstm_rows --no-cpu-baseline > gpurun_out/fin/lstm_rows_w4.json 2> gpurun_out/fin/lstm_rows_w4.err
tail -c 600 gpurun_out/fin/ours_w4.json
