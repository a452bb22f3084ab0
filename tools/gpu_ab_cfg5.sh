# cfg5 (R-MAT s22 k-truss support) multiply time with library variants: phase split (profile_cfg, 3 reps).
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then lib=paper_2111_09947_b200/_lib/libmaskmul_b200.so; else lib=tools/_variants/lib_$v.so; fi
  echo "== $v"; MM_LIB_PATH=$lib timeout 600 python tools/profile_cfg.py cfg5 auto 3 2>&1 | tail -1 | cut -c1-200
done
