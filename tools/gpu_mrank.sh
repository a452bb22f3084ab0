# Multi-rank plumbing check on ONE GPU: 2 ranks over gloo on cuda:0 (no data-path
# collective: the ranks never wait on each other inside a kernel).  Not a measurement.
mkdir -p gpurun_out
MM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mrank.json 2> gpurun_out/mrank.err; echo mrank rc=$?
MM_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/mrank_ref.json 2> gpurun_out/mrank_ref.err; echo mrank_ref rc=$?
cat gpurun_out/mrank.json; tail -5 gpurun_out/mrank.err
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench1 rc=$?
