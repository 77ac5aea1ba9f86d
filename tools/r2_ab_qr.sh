python paper_2110_02140_b200/build.py > /dev/null 2>&1
S2_DECODE_QR=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/qr_pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/qr_pytest.log
mkdir -p gpurun_out/abqr
for c in resnet50 resnet50_d4 resnet50_d8; do
  for i in 1 2; do
    for v in 1 2 3; do
      S2_DECODE_QR=$v timeout 300 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/abqr/qr${v}_${c}_$i.json 2>/dev/null
    done
  done
done
python tools/bsum.py gpurun_out/abqr/*.json
