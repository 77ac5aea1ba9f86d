# push vs pull exchange A/B at W = 2 and 4 (alternating, one box), parity of both on 4 GPUs,
# exchange phase traces, and the fixed atomics/gather microbenchmark
OUT=gpurun_out/r2_push
mkdir -p $OUT
python paper_2110_02140_b200/build.py > /dev/null 2>&1
./tools/atomics_bench > $OUT/atomics_bench3.json 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_local_ranks.py -q -p no:cacheprovider > $OUT/pytest_multi.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_multi.log
for W in 2 4; do
  for rep in 1 2; do
    for P in 0 1; do
      S2_P2P_PUSH=$P timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
        --master-port $((29700 + W * 10 + rep * 2 + P)) bench.py --gpus $W --steps 200 --no-cpu-baseline > $OUT/w${W}_push${P}_$rep.json 2> $OUT/w${W}_push${P}_$rep.err
    done
  done
  for P in 0 1; do
    S2_P2P_PUSH=$P S2_P2P_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
      --master-port $((29760 + W * 2 + P)) tools/p2p_trace.py > $OUT/trace_w${W}_push$P.json 2> $OUT/trace_w${W}_push$P.err
  done
done
tail -n 3 $OUT/pytest_multi.log
python tools/bsum.py $OUT/w*.json
grep -h "^{" $OUT/trace_*.json
cat $OUT/atomics_bench3.json
