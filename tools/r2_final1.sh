# final single-GPU evidence: smoke, full pytest -m gpu, default bench (with the CPU baseline), the
# reference arm, the launch list of the default bench, ncu --set full of compress / decode
set -x
OUT=gpurun_out/final1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo smoke_rc=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_1gpu.log 2>&1; echo pytest_rc=$?
tail -2 $OUT/pytest_gpu_1gpu.log
python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo bench_rc=$?
python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench_resnet50_w1.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_compress -s 4 -c 1 -o $OUT/compress_resnet50 -f python tools/prof_reduce.py --config resnet50 --steps 6 > $OUT/ncu_c.log 2>&1
$NCU -k regex:k_decode -s 4 -c 1 -o $OUT/decode_resnet50 -f python tools/prof_reduce.py --config resnet50 --steps 6 > $OUT/ncu_d.log 2>&1
$NCU -k regex:k_decode -s 4 -c 1 -o $OUT/decode_resnet50_d8 -f python tools/prof_reduce.py --config resnet50_d8 --steps 6 > $OUT/ncu_d8.log 2>&1
for r in compress_resnet50 decode_resnet50 decode_resnet50_d8; do ncu -i $OUT/$r.ncu-rep --page raw --csv > $OUT/${r}_raw.csv; done
ls -la $OUT
