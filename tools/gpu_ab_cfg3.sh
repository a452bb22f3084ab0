# cfg3 d16/d64 auto with library variants (bench_configs, 3 rounds each, interleaved)
for r in 1 2 3; do
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then lib=paper_2111_09947_b200/_lib/libmaskmul_b200.so; else lib=tools/_variants/lib_$v.so; fi
  MM_LIB_PATH=$lib timeout 600 python tools/bench_configs.py --configs cfg3_d16,cfg3_d64 --out gpurun_out/abc3_$v.json > /dev/null 2>&1
  python -c "
import json
print('$v', ' '.join(f\"{l['config']}:{l['gpu_ms_min']:.3f}\" for l in json.load(open('gpurun_out/abc3_$v.json')) if l['algorithm']=='auto'))"
done; done
