# A/B of library variants on cfg2: bench numeric phase + per-kernel ncu launch durations (serialized).
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2111_09947_b200/_lib/libmaskmul_b200.so; else lib=tools/_variants/lib_$v.so; fi
  for rep in 1 2; do
    MM_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/ab_$v.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['phase_ms'].items()})"
  done
  MM_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/abk_$v.csv python tools/profile_step.py --reps 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/abk_$v.csv 9
done
