# GPU call: cfg3 d16/d64 phase split + launch lists (where do the 0.7-0.8 ms go)
mkdir -p gpurun_out
for d in cfg3_d16 cfg3_d64; do
  timeout 300 python tools/profile_cfg.py $d auto 5 > gpurun_out/phase_$d.log 2>&1; echo $d rc=$?
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$d.csv python tools/profile_cfg.py $d auto 1 > /dev/null 2>&1; echo ncu $d rc=$?
done
cat gpurun_out/phase_cfg3_d16.log gpurun_out/phase_cfg3_d64.log
