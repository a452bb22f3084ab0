# Boundary between the 4-warp and 16-warp tiers for plain order-free hash rows (mm_set_tuning
# param 22; param 1 sets both): cfg2 numeric phase, cfg5, then the GPU suite and BC / k-truss.
mkdir -p gpurun_out
P22="-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1:-1"
ALGOS=auto,hash TUNINGS="$P22:65536,$P22:524288,$P22:65536,$P22:524288" timeout 600 python tools/algo_sweep.py 2>&1 | cut -c140-260
rm -f gpurun_out/ab_cfg5.jsonl
for t in 65536 524288 262144; do
  TUNE="$P22:$t" REPS=2 timeout 600 python tools/ab_cfg5.py >> gpurun_out/ab_cfg5.jsonl 2>> gpurun_out/ab_cfg5.err; echo hash tier1=$t rc=$?
done
cut -c70-200 gpurun_out/ab_cfg5.jsonl
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider 2>&1 | tail -2
timeout 600 python tools/bench_bc.py 2>/dev/null | cut -c1-200
timeout 600 python tools/bench_ktruss.py --scale 18 2>/dev/null | cut -c1-200
timeout 600 python tools/bench_configs.py --configs cfg1,cfg3_d16,cfg4 2>/dev/null | grep '"auto"' | cut -c1-110
