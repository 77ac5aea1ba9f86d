# ncu --set full of the decode at the W=8-union proxy and the headline; raw metric dumps for the l1tex breakdown
set -x
python paper_2110_02140_b200/build.py > /dev/null 2>&1
python tools/prof_reduce.py --config resnet50_d8 --steps 6 || exit 1
NCU="ncu --set full --import-source on --clock-control none"
for c in resnet50_d8 resnet50_d4; do
$NCU -k regex:k_decode -s 4 -c 1 -o gpurun_out/dec_$c -f python tools/prof_reduce.py --config $c --steps 6 > gpurun_out/ncu_dec_$c.log 2>&1
ncu -i gpurun_out/dec_$c.ncu-rep --page raw --csv > gpurun_out/dec_${c}_raw.csv
ncu -i gpurun_out/dec_$c.ncu-rep --page details --csv > gpurun_out/dec_${c}_details.csv
done
