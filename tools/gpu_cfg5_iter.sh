# cfg5 iteration: sliced-row tests + golden, then variants' cfg5 time.
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "search_mode or cfg5 or every_tier" > gpurun_out/cfg5_iter_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/cfg5_iter_tests.log
MM_LIB_PATH=tools/_variants/lib_w8m2.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "search_mode or cfg5" > gpurun_out/cfg5_iter_tests_w8.log 2>&1; echo tests w8m2 rc=$?; tail -1 gpurun_out/cfg5_iter_tests_w8.log
VARIANTS="base w8m2" bash tools/gpu_ab_cfg5.sh
echo "== base, no cursors"; TUNE=0:0:0:0:0:0:0:-1:-1:-1:-1:0:-1:-1:-1:0 timeout 600 python tools/profile_cfg.py cfg5 auto 3 2>&1 | tail -1 | cut -c1-120
