# decode two-query batching A/B (ab/old = HEAD without it) + atomics microbenchmark + sanitizer runs
bash tools/ab_run.sh "resnet50 resnet50_d4 resnet50_d8" 2 > gpurun_out/r2_ab_dec.txt 2>&1
./tools/atomics_bench > gpurun_out/r2_atomics_bench.json 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
$CS --tool memcheck --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/r2_sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2_sanitizer_memcheck.log
$CS --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/r2_sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/r2_sanitizer_racecheck.log
$CS --tool synccheck --error-exitcode 9 python tools/sanitize_probe.py > gpurun_out/r2_sanitizer_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/r2_sanitizer_synccheck.log
timeout 600 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_probe.py --local 2 > gpurun_out/r2_sanitizer_memcheck_local2.log 2>&1; echo "memcheck local2 rc=$?" >> gpurun_out/r2_sanitizer_memcheck_local2.log
tail -3 gpurun_out/r2_sanitizer_*.log
cat gpurun_out/r2_ab_dec.txt gpurun_out/r2_atomics_bench.json
