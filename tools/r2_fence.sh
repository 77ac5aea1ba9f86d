python paper_2110_02140_b200/build.py >/dev/null 2>&1
timeout 900 python -m pytest tests/test_local_ranks.py tests/test_gpu_parity.py -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2; do python bench.py --config resnet50 --steps 300 --no-cpu-baseline > gpurun_out/fence_w1_$i.json 2>/dev/null; done
for W in 2 4; do for i in 1 2; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29900+W*10+i)) bench.py --gpus $W --steps 200 > gpurun_out/fence_w${W}_$i.json 2>/dev/null; done; done
python tools/bsum.py gpurun_out/fence_*.json
