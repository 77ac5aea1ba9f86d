# A/B of two prebuilt libraries (ab/libs2_base.so vs ab/libs2_var.so), alternating: bash tools/ab_lib.sh "<configs>" [reps]
mkdir -p gpurun_out/ablib
CFGS=${1:-resnet50}
REPS=${2:-2}
for c in $CFGS; do
  for i in $(seq 1 $REPS); do
    S2_LIB=ab/libs2_base.so timeout 300 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/ablib/base_${c}_$i.json 2>/dev/null
    S2_LIB=ab/libs2_var.so timeout 300 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/ablib/var_${c}_$i.json 2>/dev/null
  done
done
python tools/bsum.py gpurun_out/ablib/*.json
