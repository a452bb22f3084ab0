# iteration: parity + acceptance + graph ops + integration stub tests, BC bench, cfg3 table
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_graph_ops.py tests/test_gpu_integration_stub.py -m gpu -q -x -p no:cacheprovider -k "not cfg5" > gpurun_out/iter2_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/iter2_tests.log
timeout 600 python tools/bench_bc.py > gpurun_out/iter2_bc.json 2>&1; echo bc rc=$?; head -c 400 gpurun_out/iter2_bc.json; echo
timeout 900 python tools/bench_configs.py --configs cfg1,cfg3_d1,cfg3_d16,cfg3_d64 --out gpurun_out/iter2_configs.json > /dev/null 2>&1; echo configs rc=$?
python - <<'P'
import json
for l in json.load(open("gpurun_out/iter2_configs.json")):
    if l["algorithm"] in ("auto", "auto+pull", "msa", "hash"): print(l["config"], l["algorithm"], round(l["gpu_ms_min"], 3), round(l["roofline_frac_measured_peak"], 3))
P
