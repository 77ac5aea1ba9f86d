# cross-reduce overlap (compress i+1 with decode i): parity suite + A/B S2_OVERLAP=0 vs default
python paper_2110_02140_b200/build.py > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_overlap_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_overlap_pytest.log
tail -n 3 gpurun_out/r2_overlap_pytest.log
bash tools/ab_env.sh "S2_OVERLAP=0" "resnet50 gpt2m_99 lstm_rows bert" 2 > gpurun_out/r2_ab_overlap.txt 2>&1
cat gpurun_out/r2_ab_overlap.txt
