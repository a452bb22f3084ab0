for r in 1 2; do
for c in fcee2e3 e593846; do
  (cd tools/_variants/wt/$c && timeout 600 python tools/bench_configs.py --configs cfg3_d16,cfg3_d64 --out /tmp/bis_$c.json > /dev/null 2>&1; python -c "
import json
print('$c', ' '.join(f\"{l['config']}:{l['gpu_ms_min']:.3f}\" for l in json.load(open('/tmp/bis_$c.json')) if l['algorithm']=='auto'))")
done
timeout 600 python tools/bench_configs.py --configs cfg3_d16,cfg3_d64 --out /tmp/bis_head.json > /dev/null 2>&1; python -c "
import json
print('HEAD', ' '.join(f\"{l['config']}:{l['gpu_ms_min']:.3f}\" for l in json.load(open('/tmp/bis_head.json')) if l['algorithm']=='auto'))"
done
