# ncu --set full of the cfg3 d16 / d64 numeric kernels (auto, push) -> CSV exports in gpurun_out/ncu/
mkdir -p gpurun_out/ncu
TAG=${TAG:-iter}
for d in ${DS:-16 64}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_push|k_pull}" -o /tmp/${TAG}_cfg3_d$d python tools/profile_cfg.py cfg3_d$d ${ALGO:-auto} 1 > gpurun_out/ncu_${TAG}_d$d.log 2>&1; echo ncu d$d rc=$?
  ncu -i /tmp/${TAG}_cfg3_d$d.ncu-rep --page raw --csv > gpurun_out/ncu/${TAG}_cfg3_d${d}_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_cfg3_d$d.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/${TAG}_cfg3_d${d}_source.csv 2>/dev/null
  gzip -f gpurun_out/ncu/${TAG}_cfg3_d${d}_source.csv
  python tools/ncu_summary.py gpurun_out/ncu/${TAG}_cfg3_d${d}_raw.csv
done
