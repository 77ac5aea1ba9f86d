mkdir -p gpurun_out/push2
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "push" > gpurun_out/push2/multigpu.log 2>&1; tail -2 gpurun_out/push2/multigpu.log
S2_P2P_PUSH_FENCE=2 timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "push" > gpurun_out/push2/multigpu_f2.log 2>&1; tail -2 gpurun_out/push2/multigpu_f2.log
for N in 2 4; do
  for i in 1 2; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --no-cpu-baseline > gpurun_out/push2/base_w${N}_$i.json 2>/dev/null
    for F in 0 1 2; do
    S2_P2P_PUSH_FENCE=$F S2_P2P_BITMAP_PUSH_MAXW=8 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N > gpurun_out/push2/push_f${F}_w${N}_$i.json 2>/dev/null
    done
  done
done
python tools/bsum.py gpurun_out/push2/*.json
