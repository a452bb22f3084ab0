# A/B of library variants on cfg2 (bench.py numeric phase), alternating runs.
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=paper_2111_09947_b200/_lib/libmaskmul_b200.so; else lib=tools/_variants/lib_$v.so; fi
    MM_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/ab_$v.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['phase_ms'].items()})"
  done
done
