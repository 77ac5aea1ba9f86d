# last measurement run of the round (4 GPUs): tests, smoke, bench W=1/2/4 + reference arm, ncu
set -x
O=gpurun_out/fin3
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt; nproc >> $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 300 python bench.py > $O/ours_w1.json 2> $O/ours_w1.err
timeout 400 python bench.py --impl reference --steps 20 --warmup 3 > $O/ref_w1.json 2> $O/ref_w1.err
for N in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N > $O/ours_w$N.json 2> $O/ours_w$N.err
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --impl reference --steps 20 --warmup 3 > $O/ref_w$N.json 2> $O/ref_w$N.err
done
bash tools/ab_multi_dist.sh 2 S2_P2P_GRID "74 296" resnet50 1
bash tools/ab_multi_dist.sh 4 S2_P2P_GRID "74 296" resnet50 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_compress|k_decode" -s 4 -c 2 -o $O/prof python tools/prof_reduce.py > $O/prof_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/launch_ncu.log 2>&1
tail -3 $O/pytest_gpu.log
python tools/bsum.py $O/*.json gpurun_out/abd/*GRID*.json
