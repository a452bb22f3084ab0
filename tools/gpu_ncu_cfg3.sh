# GPU call: ncu --set full of the cfg3 d16 numeric kernel (MCA tier 0, ordered float64)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_push' -o gpurun_out/cfg3_d16 python tools/profile_cfg.py cfg3_d16 auto 1 > gpurun_out/ncu_cfg3.log 2>&1; echo ncu rc=$?
ls -la gpurun_out/cfg3_d16.ncu-rep
