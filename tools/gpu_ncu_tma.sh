# ncu --set full of the dominant cfg2 kernel (k_push_rank<4,...>) in the base build and the TMA-staging variant.
mkdir -p gpurun_out/ncu
for v in base tma256; do
  if [ $v = base ]; then lib=paper_2111_09947_b200/_lib/libmaskmul_b200.so; else lib=tools/_variants/lib_$v.so; fi
  MM_LIB_PATH=$lib timeout 600 ncu --set full --clock-control none -k regex:k_push_rank --launch-count 1 -o /tmp/tma_$v python tools/profile_step.py --reps 1 > gpurun_out/ncu_tma_$v.log 2>&1; echo "$v rc=$?"
  ncu -i /tmp/tma_$v.ncu-rep --page raw --csv > gpurun_out/ncu/r2_tma_${v}_rank4_raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/ncu/r2_tma_${v}_rank4_raw.csv
done
