# bash tools/ab_multi.sh VAR "v1 v2 ..." "<configs>" [reps]   (v = "" runs without VAR)
mkdir -p gpurun_out/abm
VAR=$1; VALS=$2; CFGS=${3:-resnet50}; REPS=${4:-2}
for c in $CFGS; do
  for i in $(seq 1 $REPS); do
    timeout 300 python bench.py --config $c --no-cpu-baseline --steps 500 > gpurun_out/abm/${c}_base_$i.json 2>/dev/null
    for v in $VALS; do
      timeout 300 env $VAR=$v python bench.py --config $c --no-cpu-baseline --steps 500 > gpurun_out/abm/${c}_${VAR}${v}_$i.json 2>/dev/null
    done
  done
done
python tools/bsum.py gpurun_out/abm/*.json
