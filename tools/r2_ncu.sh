# ncu captures for round 2 (1 GPU): full set + source counters of compress/decode at the headline
# config and the W=8-union decode proxy; launch list of the default bench.  Outputs in gpurun_out/.
set -x
python paper_2110_02140_b200/build.py > /dev/null 2>&1
python tools/prof_reduce.py --config resnet50 --steps 6 || exit 1
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_compress -s 4 -c 1 -o gpurun_out/r2_compress_resnet50 -f python tools/prof_reduce.py --config resnet50 --steps 6 > gpurun_out/r2_ncu_c.log 2>&1
$NCU -k regex:k_decode -s 4 -c 1 -o gpurun_out/r2_decode_resnet50 -f python tools/prof_reduce.py --config resnet50 --steps 6 > gpurun_out/r2_ncu_d.log 2>&1
$NCU -k regex:k_decode -s 4 -c 1 -o gpurun_out/r2_decode_resnet50_d8 -f python tools/prof_reduce.py --config resnet50_d8 --steps 6 > gpurun_out/r2_ncu_d8.log 2>&1
$NCU -k regex:k_compress -s 4 -c 1 -o gpurun_out/r2_compress_resnet50_d8 -f python tools/prof_reduce.py --config resnet50_d8 --steps 6 > gpurun_out/r2_ncu_c8.log 2>&1
for c in resnet50 resnet50_d4 resnet50_d8; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench_$c.json 2>gpurun_out/r2_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_resnet50.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
