mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python tools/ab_cfg5.py > gpurun_out/cfg5_default.json 2>&1; echo cfg5 rc=$?
timeout 900 python tools/bench_ktruss.py --scale 22 > gpurun_out/ktruss_s22.json 2> gpurun_out/ktruss_s22.err; echo k22 rc=$?
timeout 900 python tools/bench_ktruss.py --scale 18 --cpu > gpurun_out/ktruss_s18.json 2> gpurun_out/ktruss_s18.err; echo k18 rc=$?
timeout 900 python tools/sanitize_smoke.py > gpurun_out/kernel_smoke.log 2>&1; echo ksmoke rc=$?
tail -1 gpurun_out/gpu_tests.log; cat gpurun_out/cfg5_default.json
