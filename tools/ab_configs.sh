# A/B of library variants (tools/_variants/lib_<name>.so) on the small configs and BC.
mkdir -p gpurun_out
for v in "$@"; do
  lib=tools/_variants/lib_$v.so
  MM_LIB_PATH=$lib timeout 900 python tools/bench_configs.py --configs ${CFGS:-cfg1,cfg3_d1,cfg3_d4,cfg3_d16,cfg3_d64,cfg4} > gpurun_out/abc_$v.jsonl 2> gpurun_out/abc_$v.err; echo $v cfg rc=$?
  MM_LIB_PATH=$lib timeout 600 python tools/bench_bc.py --reps 3 > gpurun_out/abbc_$v.json 2>> gpurun_out/abc_$v.err; echo $v bc rc=$?
done
