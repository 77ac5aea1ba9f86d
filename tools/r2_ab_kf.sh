# A/B: compress tile KF=8 vs KF=4, and the decode two-query batching (resnet50 d1/d4/d8)
python paper_2110_02140_b200/build.py > /dev/null 2>&1
for kf in 8 4; do
  for c in resnet50 resnet50_d4 resnet50_d8; do
    S2_COMPRESS_KF=$kf python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('kf=$kf', '$c', d['ms_per_step'], {k:v['ms'] for k,v in d['phases'].items()})"
  done
  S2_COMPRESS_KF=$kf python tools/overlap_probe.py 0.01
done
S2_COMPRESS_KF=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -p no:cacheprovider 2>&1 | tail -2
