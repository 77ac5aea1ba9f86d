# exchange CTA size / grid under the two-stream pipeline (W = 2, 4)
python paper_2110_02140_b200/build.py >/dev/null 2>&1
mkdir -p gpurun_out/abx
for W in 4 2; do
  for tg in 1024:0 512:0 256:0 512:148 256:148 1024:0; do
    t=${tg%%:*}; g=${tg##*:}
    if [ $g = 0 ]; then GE=""; else GE="S2_P2P_GRID=$g"; fi
    env S2_P2P_THREADS=$t $GE timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
      --master-port $((29800 + W + t/16 + g)) bench.py --gpus $W --steps 200 > gpurun_out/abx/w${W}_t${t}_g${g}_$(date +%s).json 2>/dev/null
  done
done
python tools/bsum.py gpurun_out/abx/*.json
