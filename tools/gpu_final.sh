# Final validation: GPU tests, smoke, bench (both arms), small-case smoke of every kernel family
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 600 python tools/sanitize_smoke.py > gpurun_out/kernel_smoke.log 2>&1; echo ksmoke rc=$?
tail -2 gpurun_out/gpu_tests.log; tail -2 gpurun_out/kernel_smoke.log
