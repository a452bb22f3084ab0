"""Sum ncu gpu__time_duration per kernel from a --csv launch list."""
import collections
import csv
import sys

agg = collections.defaultdict(float)
cnt = collections.Counter()
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"][:100]
            agg[k] += float(d["Metric Value"].replace(",", ""))
            cnt[k] += 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"{v / 1e3:9.1f} us  x{cnt[k]:<3d} {k}")
