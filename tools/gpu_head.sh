# Quick HEAD check on one B200: GPU tests, smoke, bench, all-config table (no CPU oracle).
mkdir -p gpurun_out
P=${PFX:-head}
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/${P}_gpu_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/${P}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo bench rc=$?; cat gpurun_out/${P}_bench.json | cut -c1-600
timeout 1500 python tools/bench_configs.py --configs cfg1,cfg2,cfg3_d1,cfg3_d4,cfg3_d16,cfg3_d64,cfg4,cfg5 --out gpurun_out/${P}_configs.json > gpurun_out/${P}_configs.log 2>&1; echo configs rc=$?; tail -30 gpurun_out/${P}_configs.log
