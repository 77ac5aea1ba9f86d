# ncu --set full of one kernel under an env switch: bash tools/r2_ncu_var.sh <tag> <kernel-regex> <config> [ENV=val ...]
TAG=$1; KR=$2; CFG=$3; shift 3
python paper_2110_02140_b200/build.py > /dev/null 2>&1
env "$@" python tools/prof_reduce.py --config $CFG --steps 6 || exit 1
env "$@" ncu --set full --import-source on --clock-control none -k regex:$KR -s 4 -c 1 -o gpurun_out/$TAG -f python tools/prof_reduce.py --config $CFG --steps 6 > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv
