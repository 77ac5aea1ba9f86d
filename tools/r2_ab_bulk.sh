# decode bulk-store variant: parity (gpu tests with the switch on) + alternating A/B at 1 % / 4 % / 7.7 % unions
python paper_2110_02140_b200/build.py > /dev/null 2>&1
S2_DECODE_BULK=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or local or bounds" > gpurun_out/bulk_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/bulk_pytest.log
bash tools/ab_env.sh "S2_DECODE_BULK=1" "resnet50 resnet50_d4 resnet50_d8" 2
