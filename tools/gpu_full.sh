# Full check on one B200: all GPU tests, smoke, bench (both arms), all configs, partition balance, 2-rank plumbing.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1500 -p no:cacheprovider > gpurun_out/full_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/full_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/full_smoke.log
timeout 600 python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/full_bench.json')); print('bench', d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['phase_ms'])"
timeout 600 python bench.py --impl reference > gpurun_out/full_bench_ref.json 2> gpurun_out/full_bench_ref.err; echo ref rc=$?
timeout 1200 python tools/bench_configs.py --configs cfg1,cfg2,cfg3_d1,cfg3_d4,cfg3_d16,cfg3_d64,cfg4,cfg5 --out gpurun_out/full_configs.json > gpurun_out/full_configs.log 2>&1; echo configs rc=$?
python - <<'P'
import json
for l in json.load(open("gpurun_out/full_configs.json")):
    print(l["config"], l["algorithm"], round(l["gpu_ms_min"], 3), round(l["roofline_frac_measured_peak"], 3))
P
bash tools/gpu_mrank.sh > gpurun_out/full_mrank.log 2>&1; echo mrank rc=$?; tail -4 gpurun_out/full_mrank.log
