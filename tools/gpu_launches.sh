# Launch lists (every kernel's device time, ncu --metrics gpu__time_duration.sum) of one multiply per config.
mkdir -p gpurun_out/launch
for spec in ${SPECS:-"cfg1 auto" "cfg3_d1 inner" "cfg3_d16 auto" "cfg4 auto"}; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch/$1_$2.csv python tools/profile_cfg.py $1 $2 2 > /dev/null 2>&1
  echo "== $1 $2"; python tools/launch_summary.py gpurun_out/launch/$1_$2.csv 2>&1 | tail -25
done
