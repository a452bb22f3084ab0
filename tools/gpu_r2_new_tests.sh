# Round-2 new GPU tests + partition balance (one B200).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_robustness.py tests/test_gpu_partition.py -m gpu -q -x -s -p no:cacheprovider > gpurun_out/r2_new_tests.log 2>&1; echo newtests rc=$?
tail -30 gpurun_out/r2_new_tests.log
timeout 1200 python tools/partition_balance.py --out gpurun_out/r2_partition_balance.json > gpurun_out/r2_partition_balance.log 2>&1; echo balance rc=$?
tail -3 gpurun_out/r2_partition_balance.log
