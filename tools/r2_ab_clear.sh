python paper_2110_02140_b200/build.py >/dev/null 2>&1
S2_DECODE_CLEAR=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py tests/test_local_ranks.py -q -p no:cacheprovider -x > gpurun_out/clear_pytest.log 2>&1; echo rc=$?; tail -2 gpurun_out/clear_pytest.log
rm -rf gpurun_out/abenv
bash tools/ab_env.sh "S2_DECODE_CLEAR=1" "resnet50 resnet50_d4 resnet50_d8 bert gpt2m_99 lstm_rows" 2
