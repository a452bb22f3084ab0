mkdir -p gpurun_out
P=${PFX:-fused}
timeout 300 python -m pytest tests/test_gpu_fused_tail.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/${P}_tail_tests.log 2>&1; echo tail rc=$?; tail -3 gpurun_out/${P}_tail_tests.log
timeout 120 python tools/py_overhead.py > gpurun_out/${P}_py_overhead.txt 2>&1; cat gpurun_out/${P}_py_overhead.txt
MM_HOST_TRACE=1 timeout 120 python tools/py_overhead.py 2>&1 | grep "mm trace" | tail -4
timeout 600 python tools/bench_configs.py --configs cfg1 --out gpurun_out/${P}_configs.json > gpurun_out/${P}_configs.log 2>&1; echo configs rc=$?; grep -h '"config"' gpurun_out/${P}_configs.log | cut -c1-130
