# ncu --set full + SASS source of cfg5's 16-warp hash launches (the first two k_push_hash launches)
mkdir -p gpurun_out/ncu
TAG=${TAG:-iter}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_push_hash --launch-count 2 -o /tmp/${TAG}_cfg5 python tools/profile_cfg.py cfg5 auto 1 > gpurun_out/ncu_${TAG}_cfg5.log 2>&1; echo ncu rc=$?
ncu -i /tmp/${TAG}_cfg5.ncu-rep --page raw --csv > gpurun_out/ncu/${TAG}_cfg5_hash16_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_cfg5.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/${TAG}_cfg5_hash16_source.csv 2>/dev/null
gzip -f gpurun_out/ncu/${TAG}_cfg5_hash16_source.csv
python tools/ncu_summary.py gpurun_out/ncu/${TAG}_cfg5_hash16_raw.csv
