# Iteration check on one B200: fp64/heap parity tests + the cfg3 / cfg4 table.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -q -x -p no:cacheprovider -k "not cfg5" > gpurun_out/iter_tests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/iter_tests.log
timeout 900 python tools/bench_configs.py --configs cfg1,cfg3_d1,cfg3_d4,cfg3_d16,cfg3_d64,cfg4 --out gpurun_out/iter_configs.json > gpurun_out/iter_configs.log 2>&1; echo configs rc=$?
python - <<'P'
import json
for l in json.load(open("gpurun_out/iter_configs.json")):
    print(l["config"], l["algorithm"], round(l["gpu_ms_min"], 3), round(l["roofline_frac_measured_peak"], 3))
P
MM_HOST_TRACE=1 timeout 300 python tools/overhead.py > gpurun_out/iter_overhead.log 2>&1; echo overhead rc=$?
grep -v "mm trace" gpurun_out/iter_overhead.log | tail; grep "mm trace" gpurun_out/iter_overhead.log | tail -3
