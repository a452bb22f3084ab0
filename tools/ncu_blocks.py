"""Group an `ncu --page source --csv --print-source sass` dump into runs of
consecutive instructions with the same execution count (≈ basic blocks) and
print the heaviest runs: share of executed instructions, share of stall
samples, first instruction."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[3] if len(sys.argv) > 3 else ""
# a dump may hold several kernels, each "Kernel Name" row followed by a header
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
for a, b in zip(starts[:-1], starts[1:]):
    if want in rows[a][1]:
        print(rows[a][1][:100])
        hdr = rows[a + 1]
        data = [r for r in rows[a + 2:b] if len(r) == len(hdr)]
        break
ix = hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ix]) for r in data)
stot = sum(int(r[st]) for r in data) or 1
runs = []
cur = None
for i, r in enumerate(data):
    n = int(r[ix])
    if cur and cur["n"] == n:
        cur["len"] += 1
        cur["st"] += int(r[st])
    else:
        cur = {"start": i, "n": n, "len": 1, "st": int(r[st]), "first": r[1].strip()[:60]}
        runs.append(cur)
runs.sort(key=lambda c: -c["n"] * c["len"])
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
acc = 0.0
for c in runs[:top]:
    share = c["n"] * c["len"] / tot * 100
    acc += share
    print(f"@{c['start']:5d} len {c['len']:4d} x {c['n']:>10d}  {share:5.1f}% (cum {acc:5.1f}%)  stall {c['st']/stot*100:5.1f}%  {c['first']}")
