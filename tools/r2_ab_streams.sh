# two-stream s2_reduce_many (exchange beside compress AND decode) vs one stream: harness parity, then W=2/4 benches
python paper_2110_02140_b200/build.py >/dev/null 2>&1
timeout 900 python -m pytest tests/test_local_ranks.py tests/test_multigpu.py -q -p no:cacheprovider -x > gpurun_out/streams_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/streams_pytest.log
mkdir -p gpurun_out/abs
for i in 1 2; do
 for W in 2 4; do
  for v in 2 1; do
    S2_PIPE_STREAMS=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
      --master-port $((29700 + W + 10*v + 100*i)) bench.py --gpus $W --steps 200 > gpurun_out/abs/s${v}_w${W}_$i.json 2> gpurun_out/abs/s${v}_w${W}_$i.err
  done
 done
done
python tools/bsum.py gpurun_out/abs/*.json
