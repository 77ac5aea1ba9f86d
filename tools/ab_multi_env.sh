# A/B/C... of an environment variable's values, alternating: bash tools/ab_multi_env.sh VAR "v1 v2 .." "<configs>" [reps]
VAR=$1; VALS=$2; CFGS=$3; REPS=${4:-2}
mkdir -p gpurun_out/abm
for c in $CFGS; do
  for i in $(seq 1 $REPS); do
    for v in $VALS; do
      env $VAR=$v timeout 300 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/abm/${VAR}${v}_${c}_$i.json 2>/dev/null
    done
  done
done
python tools/bsum.py gpurun_out/abm/*.json
