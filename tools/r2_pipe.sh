# pipelined batches (s2_reduce_many): parity on 4 GPUs + harness, A/B --pipeline 4 vs 1 at W = 2 / 4
OUT=gpurun_out/r2_pipe
mkdir -p $OUT
python paper_2110_02140_b200/build.py > /dev/null 2>&1
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_4gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_4gpu.log
tail -n 4 $OUT/pytest_gpu_4gpu.log
for W in 2 4; do
  for rep in 1 2; do
    for P in 1 4 8; do
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
        --master-port $((29800 + W * 20 + rep * 4 + P)) bench.py --gpus $W --steps 200 --pipeline $P --no-cpu-baseline > $OUT/w${W}_p${P}_$rep.json 2> $OUT/w${W}_p${P}_$rep.err
    done
  done
done
python tools/bsum.py $OUT/w*.json
