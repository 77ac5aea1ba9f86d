# bash tools/ab_multi_dist.sh N VAR "v1 v2" [config] [reps] — torchrun A/B of an env switch at N GPUs
mkdir -p gpurun_out/abd
N=$1; VAR=$2; VALS=$3; C=${4:-resnet50}; REPS=${5:-2}
for i in $(seq 1 $REPS); do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus $N --config $C > gpurun_out/abd/w${N}_${C}_base_$i.json 2>/dev/null
  for v in $VALS; do
    timeout 300 env $VAR=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus $N --config $C > gpurun_out/abd/w${N}_${C}_${VAR}${v}_$i.json 2>/dev/null
  done
done
