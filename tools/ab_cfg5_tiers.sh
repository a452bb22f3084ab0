# cfg5: 4-warp / 16-warp tier boundary (mm_set_tuning param 1) and the slice size variant
mkdir -p gpurun_out
for t in 32768 131072 262144 1048576; do
  TUNE="-1:$t" REPS=2 timeout 600 python tools/ab_cfg5.py >> gpurun_out/ab_cfg5.jsonl 2>> gpurun_out/ab_cfg5.err; echo tier1=$t rc=$?
done
bash tools/ab_cfg5.sh base slice4 > /dev/null
cut -c1-200 gpurun_out/ab_cfg5.jsonl
