# Per-kernel launch times (ncu launch list) of library variants on one cfg2 multiply.
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2111_09947_b200/_lib/libmaskmul_b200.so; else lib=tools/_variants/lib_$v.so; fi
  MM_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kl_$v.csv python tools/profile_step.py --reps 2 > /dev/null 2>&1
  echo "== $v"; python tools/launch_summary.py gpurun_out/kl_$v.csv | grep "k_push\|k_pull" | head -10
done
