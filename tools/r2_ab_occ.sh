# A/B compress occupancy (S2_COMPRESS_OCC=3: 80 registers, 3 CTAs/SM) + gather/atomic microbench + bounds tests
python paper_2110_02140_b200/build.py > /dev/null 2>&1
bash tools/ab_env.sh "S2_COMPRESS_OCC=3" "resnet50 gpt2m_99" 2 > gpurun_out/r2_ab_occ.txt 2>&1
for o in 2 3; do S2_COMPRESS_OCC=$o python tools/overlap_probe.py 0.01 >> gpurun_out/r2_ab_occ.txt 2>&1; done
./tools/atomics_bench > gpurun_out/r2_atomics_bench2.json 2>&1
timeout 900 python -m pytest tests/test_gpu_bounds.py -q -p no:cacheprovider > gpurun_out/r2_bounds.log 2>&1; echo "bounds rc=$?" >> gpurun_out/r2_bounds.log
S2_COMPRESS_OCC=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "golden or random_shapes or full_size" > gpurun_out/r2_occ3_parity.log 2>&1; echo "occ3 parity rc=$?" >> gpurun_out/r2_occ3_parity.log
cat gpurun_out/r2_ab_occ.txt; tail -3 gpurun_out/r2_bounds.log gpurun_out/r2_occ3_parity.log; cat gpurun_out/r2_atomics_bench2.json
