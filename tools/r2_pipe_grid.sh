# exchange grid under pipelining (fewer exchange CTAs leave more SMs to the overlapping compress)
OUT=gpurun_out/r2_pipe_grid
mkdir -p $OUT
python paper_2110_02140_b200/build.py > /dev/null 2>&1
for W in 2 4; do
  for rep in 1 2; do
    for G in 0 37 24; do
      if [ $G -eq 0 ]; then ENVG=""; else ENVG="S2_P2P_GRID=$G"; fi
      env $ENVG timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
        --master-port $((29900 + W * 20 + rep * 4 + G % 7)) bench.py --gpus $W --steps 200 --no-cpu-baseline > $OUT/w${W}_g${G}_$rep.json 2> $OUT/w${W}_g${G}_$rep.err
    done
  done
done
python tools/bsum.py $OUT/w*.json
