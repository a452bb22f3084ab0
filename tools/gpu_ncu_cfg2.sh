# ncu --set full + SASS source pages of the cfg2 numeric kernels -> gpurun_out/ncu/${TAG}_cfg2_*
mkdir -p gpurun_out/ncu
TAG=${TAG:-iter}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_push|k_pull}" -o /tmp/${TAG}_cfg2 python tools/profile_step.py --reps 1 > gpurun_out/ncu_${TAG}_cfg2.log 2>&1; echo ncu rc=$?
ncu -i /tmp/${TAG}_cfg2.ncu-rep --page raw --csv > gpurun_out/ncu/${TAG}_cfg2_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_cfg2.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/${TAG}_cfg2_source.csv 2>/dev/null
gzip -f gpurun_out/ncu/${TAG}_cfg2_source.csv
python tools/ncu_summary.py gpurun_out/ncu/${TAG}_cfg2_raw.csv
