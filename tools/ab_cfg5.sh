# cfg5 A/B over library variants (tools/_variants/lib_<name>.so)
mkdir -p gpurun_out
for v in "$@"; do
  MM_LIB_PATH=tools/_variants/lib_$v.so timeout 600 python tools/ab_cfg5.py >> gpurun_out/ab_cfg5.jsonl 2>> gpurun_out/ab_cfg5.err; echo $v rc=$?
done
cat gpurun_out/ab_cfg5.jsonl
