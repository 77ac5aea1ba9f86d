# A/B of an environment switch on one box, alternating: bash tools/ab_env.sh "VAR=val" "<configs>" [reps]
mkdir -p gpurun_out/abenv
ENVSET=$1
CFGS=${2:-resnet50}
REPS=${3:-3}
for c in $CFGS; do
  for i in $(seq 1 $REPS); do
    timeout 300 python bench.py --config $c --no-cpu-baseline --steps 500 > gpurun_out/abenv/base_${c}_$i.json 2>/dev/null
    timeout 300 env $ENVSET python bench.py --config $c --no-cpu-baseline --steps 500 > gpurun_out/abenv/var_${c}_$i.json 2>/dev/null
  done
done
python tools/bsum.py gpurun_out/abenv/*.json
