for c in ae90169 038330c 3c47b08 8abd48d; do
  (cd tools/_variants/wt/$c && timeout 600 python tools/bench_bc.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$c', round(d['gpu_seconds_wall'],3), round(d['multiply_seconds'],3))")
done
timeout 600 python tools/bench_bc.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('HEAD', round(d['gpu_seconds_wall'],3), round(d['multiply_seconds'],3))"
