timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
ALGOS=${ALGOS:-hash,msa,mca,auto} timeout 600 python tools/algo_sweep.py > gpurun_out/algo_sweep.log 2>&1; echo sweep rc=$?
