# Full round-2 evidence on one B200 (outputs gpurun_out/${P}_*; copied to profiles/r2/ afterwards):
# GPU tests, smoke, bench (both arms), launch list, ncu numeric kernels (traffic), all-config table
# with the CPU oracle, partition balance, BC / k-truss / prep / mmio benches.
mkdir -p gpurun_out
C=${COMMIT:-unknown}
P=${PFX:-r2e}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${P}_nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/${P}_gpu_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${P}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/${P}_bench_ref.json 2> gpurun_out/${P}_bench_ref.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${P}_ncu_launch.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none -k regex:'k_push|k_pull' --csv --page raw \
  python tools/profile_step.py --reps 1 > gpurun_out/${P}_ncu_full_raw.csv 2> gpurun_out/${P}_ncu_full.err; echo ncu_full rc=$?
python tools/ncu_traffic.py gpurun_out/${P}_ncu_full_raw.csv gpurun_out/${P}_ncu_traffic.json $C
timeout 1500 python tools/bench_configs.py --cpu --configs cfg1,cfg2,cfg3_d1,cfg3_d4,cfg3_d16,cfg3_d64,cfg4 --out gpurun_out/${P}_configs_cpu.json > gpurun_out/${P}_configs.log 2>&1; echo configs rc=$?
timeout 900 python tools/bench_configs.py --configs cfg5 --out gpurun_out/${P}_cfg5.json > gpurun_out/${P}_cfg5.log 2>&1; echo cfg5 rc=$?
timeout 1500 python tools/partition_balance.py --out gpurun_out/${P}_partition_balance.json > gpurun_out/${P}_partition_balance.log 2>&1; echo balance rc=$?
timeout 600 python tools/bench_bc.py --cpu > gpurun_out/${P}_bench_bc.json 2> gpurun_out/${P}_bench_bc.err; echo bc rc=$?
timeout 900 python tools/bench_ktruss.py --scale 18 --cpu > gpurun_out/${P}_ktruss_s18.json 2> gpurun_out/${P}_ktruss_s18.err; echo k18 rc=$?
timeout 900 python tools/bench_ktruss.py --scale 22 > gpurun_out/${P}_ktruss_s22.json 2> gpurun_out/${P}_ktruss_s22.err; echo k22 rc=$?
timeout 600 python tools/bench_prep.py > gpurun_out/${P}_bench_prep.json 2> gpurun_out/${P}_bench_prep.err; echo prep rc=$?
timeout 600 python tools/bench_mmio.py > gpurun_out/${P}_bench_mmio.json 2> gpurun_out/${P}_bench_mmio.err; echo mmio rc=$?
python tools/py_overhead.py > gpurun_out/${P}_py_overhead.txt 2>&1; echo overhead rc=$?
bash tools/gpu_mrank.sh > gpurun_out/${P}_mrank.log 2>&1; cp gpurun_out/mrank.json gpurun_out/${P}_mrank.json; echo mrank rc=$?
du -sh gpurun_out
