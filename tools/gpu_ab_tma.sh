# TMA-staging experiment: correctness (parity tests + bench triangles) and per-kernel time vs base on cfg2.
mkdir -p gpurun_out
for v in tma256 tma tma512min512; do
  MM_LIB_PATH=tools/_variants/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "random_cases or cfg2_triangle or every_tier" > gpurun_out/ab_tma_tests_$v.log 2>&1; echo "$v tests rc=$?"; tail -1 gpurun_out/ab_tma_tests_$v.log
done
for v in base tma256 tma tma512min512; do
  if [ $v = base ]; then lib=paper_2111_09947_b200/_lib/libmaskmul_b200.so; else lib=tools/_variants/lib_$v.so; fi
  for r in 1 2; do MM_LIB_PATH=$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_tma_bench_${v}_$r.json 2>/dev/null; done
  python -c "
import json
for r in (1,2):
    d=json.load(open('gpurun_out/ab_tma_bench_${v}_%d.json'%r)); print('$v', r, 'ms', round(d['ms_per_step'],3), 'numeric', round(d['phase_ms']['numeric'],3), 'tri_ok', d['details']['triangles_ok'])"
done
bash tools/ab_kernels.sh base tma256 tma 2>&1 | tail -40
