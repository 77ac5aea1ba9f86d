# round-2 multi-GPU evidence (run with gpurun --gpus N, N = 2 or 4): full pytest -m gpu (the
# multi-GPU tests run for W <= N), bench at W = 1..N with NVLink byte counters around each
# multi-GPU bench, the in-kernel exchange phase trace, and the CPU reference arm.
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2_multi
mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_${N}gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_${N}gpu.log
tail -3 $OUT/pytest_gpu_${N}gpu.log
for W in $(seq 1 $N); do
  [ $W -eq 3 ] && continue
  nvidia-smi nvlink -gt d > $OUT/nvlink_before_w$W.txt 2>&1
  if [ $W -eq 1 ]; then
    timeout 600 python bench.py --gpus 1 > $OUT/ours_w1.json 2> $OUT/ours_w1.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
      --master-port $((29600 + W)) bench.py --gpus $W > $OUT/ours_w$W.json 2> $OUT/ours_w$W.err
  fi
  nvidia-smi nvlink -gt d > $OUT/nvlink_after_w$W.txt 2>&1
  if [ $W -gt 1 ]; then
    S2_P2P_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
      --master-port $((29620 + W)) tools/p2p_trace.py > $OUT/p2p_trace_w$W.json 2> $OUT/p2p_trace_w$W.err
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
      --master-port $((29640 + W)) bench.py --gpus $W --impl reference --steps 20 --warmup 3 > $OUT/ref_w$W.json 2> $OUT/ref_w$W.err
  fi
done
timeout 600 python bench.py --gpus 1 --impl reference --steps 20 --warmup 3 > $OUT/ref_w1.json 2> $OUT/ref_w1.err
python tools/bsum.py $OUT/ours_w*.json
