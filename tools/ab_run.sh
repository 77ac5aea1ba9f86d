# A/B: ab/old (baseline tree) vs the working tree, alternating on one box
# usage: bash tools/ab_run.sh "<config list>" [reps]
mkdir -p gpurun_out/ab
CFGS=${1:-resnet50}
REPS=${2:-3}
for c in $CFGS; do
  for i in $(seq 1 $REPS); do
    (cd ab/old && timeout 300 python bench.py --config $c --no-cpu-baseline --steps 500 > ../../gpurun_out/ab/old_${c}_$i.json 2>/dev/null)
    timeout 300 python bench.py --config $c --no-cpu-baseline --steps 500 > gpurun_out/ab/new_${c}_$i.json 2>/dev/null
  done
done
python tools/bsum.py gpurun_out/ab/*.json
