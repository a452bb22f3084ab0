# GPU call: cfg5 phase split + launch list
mkdir -p gpurun_out
timeout 600 python tools/profile_cfg.py cfg5 auto 2 > gpurun_out/phase_cfg5.log 2>&1; echo cfg5 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_cfg5.csv -k regex:'k_push|k_pull|k_analyze|k_compact|k_scan' python tools/profile_cfg.py cfg5 auto 1 > /dev/null 2>&1; echo ncu rc=$?
cat gpurun_out/phase_cfg5.log
