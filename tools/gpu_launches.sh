# Launch lists (every kernel's device time, ncu --metrics gpu__time_duration.sum) of one multiply per config.
# SPECS="cfg1:auto cfg3_d1:inner ..." (config:algorithm), profile_cfg.py with REPS multiplies (default 1)
mkdir -p gpurun_out/launch
for spec in ${SPECS:-cfg1:auto cfg3_d1:inner cfg3_d16:auto cfg4:auto}; do
  c=${spec%%:*}; a=${spec#*:}
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch/${c}_$a.csv python tools/profile_cfg.py $c $a ${REPS:-1} > /dev/null 2>&1
  echo "== $c $a"; python tools/launch_summary.py gpurun_out/launch/${c}_$a.csv 2>&1 | grep "mm::" | head -20
done
