# Round-2 baseline on one B200 (before any round-2 change): every config with the
# CPU oracle beside it, and ncu --set full of cfg3 (d1 pull, d16/d64 push) and cfg5's sliced launch.
# Reports are exported to CSV on the box (raw + details pages) and the .ncu-rep files dropped.
mkdir -p gpurun_out/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python tools/bench_configs.py --cpu --configs cfg1,cfg2,cfg3_d1,cfg3_d4,cfg3_d16,cfg3_d64,cfg4 --out gpurun_out/r2_base_configs_cpu.json > gpurun_out/r2_base_configs.log 2>&1; echo configs rc=$?
timeout 900 python tools/bench_configs.py --configs cfg5 --out gpurun_out/r2_base_cfg5.json > gpurun_out/r2_base_cfg5.log 2>&1; echo cfg5 rc=$?
exp() {  # $1 = report stem
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/ncu/$1_details.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/$1_source.csv 2>/dev/null
  gzip -f gpurun_out/ncu/$1_source.csv
  ls -la gpurun_out/ncu/$1_*
}
for d in 1 16 64; do
  a=auto; [ $d = 1 ] && a=inner
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_push|k_pull' -o /tmp/r2_base_cfg3_d$d python tools/profile_cfg.py cfg3_d$d $a 1 > gpurun_out/ncu_cfg3_d$d.log 2>&1; echo ncu d$d rc=$?
  exp r2_base_cfg3_d$d
done
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_push_hash --launch-skip 2 --launch-count 1 -o /tmp/r2_base_cfg5_sliced python tools/profile_cfg.py cfg5 auto 1 > gpurun_out/ncu_cfg5.log 2>&1; echo ncu cfg5 rc=$?
exp r2_base_cfg5_sliced
du -sh gpurun_out
