# GPU call: ncu --set full of cfg5's third 16-warp hash launch (the sliced tier-3 bin)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_push_hash --launch-skip 2 --launch-count 1 -o gpurun_out/cfg5_sliced python tools/profile_cfg.py cfg5 auto 1 > gpurun_out/ncu_cfg5.log 2>&1; echo ncu rc=$?
tail -5 gpurun_out/ncu_cfg5.log
