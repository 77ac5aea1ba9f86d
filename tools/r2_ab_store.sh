python paper_2110_02140_b200/build.py >/dev/null 2>&1
timeout 600 python -m pytest tests/test_local_ranks.py -q -p no:cacheprovider -k concurrent > gpurun_out/conc.log 2>&1; echo rc=$?; tail -3 gpurun_out/conc.log
for c in resnet50 resnet50_d8 bert; do python bench.py --config $c --steps 100 --no-cpu-baseline > gpurun_out/fl_$c.json 2>gpurun_out/fl_$c.err; done
mkdir -p gpurun_out/abst
for c in resnet50 resnet50_d4 gpt2m_99; do
  for i in 1 2; do
    for v in 0 1 2; do
      S2_DECODE_STORE=$v timeout 300 python bench.py --config $c --no-cpu-baseline --steps 300 > gpurun_out/abst/st${v}_${c}_$i.json 2>/dev/null
    done
  done
done
python tools/bsum.py gpurun_out/abst/*.json
