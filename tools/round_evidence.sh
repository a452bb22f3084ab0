# Full round evidence on one B200: GPU tests, smoke, bench (both arms), launch list,
# ncu --set full of the numeric kernels (traffic), all-config table, BC bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_push|k_pull' --csv --page raw \
  python tools/profile_step.py --reps 1 > gpurun_out/ncu_full_raw.csv 2> gpurun_out/ncu_full.err; echo ncu_full rc=$?
timeout 1200 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo configs rc=$?
timeout 600 python tools/bench_bc.py --cpu > gpurun_out/bench_bc.json 2> gpurun_out/bench_bc.err; echo bc rc=$?
timeout 900 python tools/bench_ktruss.py --scale 18 --cpu > gpurun_out/ktruss_s18.json 2> gpurun_out/ktruss_s18.err; echo k18 rc=$?
timeout 900 python tools/bench_ktruss.py --scale 22 > gpurun_out/ktruss_s22.json 2> gpurun_out/ktruss_s22.err; echo k22 rc=$?
