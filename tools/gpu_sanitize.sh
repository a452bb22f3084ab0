# compute-sanitizer memcheck / racecheck over the small multiplies of every kernel family
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/memcheck.log 2>&1; echo memcheck rc=$?
tail -4 gpurun_out/memcheck.log
