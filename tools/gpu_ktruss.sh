# GPU call: graph-driver tests + full k-truss benchmarks (s18 with the CPU oracle check, s22 device only)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph_ops.py tests/test_gpu_prep.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_graph.log 2>&1; echo graph rc=$?
timeout 900 python tools/bench_ktruss.py --scale 18 --cpu > gpurun_out/ktruss_s18.json 2> gpurun_out/ktruss_s18.err; echo k18 rc=$?
timeout 900 python tools/bench_ktruss.py --scale 22 > gpurun_out/ktruss_s22.json 2> gpurun_out/ktruss_s22.err; echo k22 rc=$?
tail -2 gpurun_out/gpu_graph.log; cat gpurun_out/ktruss_s18.json gpurun_out/ktruss_s22.json; tail -3 gpurun_out/ktruss_s22.err
