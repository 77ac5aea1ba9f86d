# decode dense-tile zero-filled stage: thresholds 0 (off) / 24 / 64 at union densities 1 / 4 / 7.7 %
python paper_2110_02140_b200/build.py > /dev/null 2>&1
for rep in 1 2; do
for c in resnet50 resnet50_d4 resnet50_d8; do
  for t in 0 24 64; do
    S2_DECODE_DENSE_MIN=$t python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('dense_min=$t', '$c', d['ms_per_step'], {k:v['ms'] for k,v in d['phases'].items()})"
  done
done
done
S2_DECODE_DENSE_MIN=24 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_local_ranks.py -q -x -p no:cacheprovider -k "golden or random_shapes or full_size or edge or block or local_exchange_parity" 2>&1 | tail -n 2
python tools/local_probe.py
CUDA_DEVICE_MAX_CONNECTIONS=32 python tools/local_probe.py
