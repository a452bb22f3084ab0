# GPU tests + small-config timings + cfg5 tier-2 hash launch under ncu --set full
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1500 -p no:cacheprovider > gpurun_out/it3_gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/it3_gpu_tests.log
timeout 600 python tools/bench_configs.py --configs cfg1,cfg4 --out gpurun_out/it3_small.json > gpurun_out/it3_small.log 2>&1; echo small rc=$?; grep -h '"auto"\|"hash"' gpurun_out/it3_small.log | cut -c1-200
python tools/py_overhead.py > gpurun_out/it3_py_overhead.txt 2>&1; cat gpurun_out/it3_py_overhead.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it3_launch_cfg1.csv python tools/profile_cfg.py cfg1 auto 3 > /dev/null 2>&1; echo ncu1 rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_push_hash<16' --launch-count 1 -o gpurun_out/it3_cfg5_t2 python tools/profile_cfg.py cfg5 auto 1 > gpurun_out/it3_ncu_cfg5.log 2>&1; echo ncu5 rc=$?
