# last measurement run of the round (4 GPUs): tests, smoke, bench W=1/2/4, ncu
set -x
O=gpurun_out/fin5
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/ours_w1.json 2> $O/ours_w1.err
for N in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N > $O/ours_w$N.json 2> $O/ours_w$N.err
done
for c in bert lstm_rows gpt2m_99; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $O/${c}_w1.json 2>/dev/null
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29560 bench.py --gpus 4 --config $c > $O/${c}_w4.json 2>/dev/null
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_compress|k_decode" -s 4 -c 2 -o $O/prof python tools/prof_reduce.py > $O/prof_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/launch_ncu.log 2>&1
tail -3 $O/pytest_gpu.log
cat $O/smoke.log
python tools/bsum.py $O/*.json
