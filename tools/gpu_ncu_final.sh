# Final-state ncu --set full captures beyond cfg2: cfg3 d1 / d4 (inner: the pull kernels),
# cfg3 d16 / d64 (auto: the deferred-hit push kernel), cfg4 (auto), cfg5's (row, slice) items kernel.
mkdir -p gpurun_out/ncu
TAG=${TAG:-r2h}
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k cfg3 --timeout 500 -p no:cacheprovider 2>&1 | tail -3
TAG=$TAG DS="1 4" ALGO=inner bash tools/gpu_ncu_cfg3.sh
TAG=$TAG DS="16 64" ALGO=auto bash tools/gpu_ncu_cfg3.sh
timeout 600 ncu --set full --clock-control none -k regex:"k_push|k_pull" -o /tmp/${TAG}_cfg4 python tools/profile_cfg.py cfg4 auto 1 > gpurun_out/ncu_${TAG}_cfg4.log 2>&1; echo ncu cfg4 rc=$?
ncu -i /tmp/${TAG}_cfg4.ncu-rep --page raw --csv > gpurun_out/ncu/${TAG}_cfg4_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/ncu/${TAG}_cfg4_raw.csv
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_push_hash_items -o /tmp/${TAG}_cfg5_items python tools/profile_cfg.py cfg5 auto 1 > gpurun_out/ncu_${TAG}_cfg5_items.log 2>&1; echo ncu items rc=$?
ncu -i /tmp/${TAG}_cfg5_items.ncu-rep --page raw --csv > gpurun_out/ncu/${TAG}_cfg5_items_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_cfg5_items.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/${TAG}_cfg5_items_source.csv 2>/dev/null
gzip -f gpurun_out/ncu/${TAG}_cfg5_items_source.csv
python tools/ncu_summary.py gpurun_out/ncu/${TAG}_cfg5_items_raw.csv
du -sh gpurun_out/ncu
