timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
ALGOS=${ALGOS:-auto} TUNINGS=${TUNINGS:-} timeout 600 python tools/algo_sweep.py > gpurun_out/algo_sweep.log 2>&1; echo sweep rc=$?
python tools/profile_step.py --reps 1 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --reps 1 > gpurun_out/ncu1.log 2>&1; echo ncu rc=$?
