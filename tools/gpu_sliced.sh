# Sliced hub rows as (row, slice) items: parity tests, cfg5 A/B (items vs sequential slices), launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sliced.py tests/test_gpu_parity.py -q -x --timeout 800 -p no:cacheprovider -k "sliced or search_mode or cfg5" > gpurun_out/sliced_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/sliced_tests.log
OFF=-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:0
for t in "" $OFF "" $OFF; do TUNE=$t REPS=3 timeout 600 python tools/ab_cfg5.py; done > gpurun_out/sliced_ab.log 2>&1; echo ab rc=$?; cat gpurun_out/sliced_ab.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_cfg5_items.csv -k regex:'k_push|k_slice' python tools/profile_cfg.py cfg5 auto 1 > /dev/null 2>&1; echo ncu rc=$?
