"""Print the hottest SASS lines of an `ncu --page source --csv --print-source sass` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
th = hdr.index("Avg. Threads Executed")
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
tot = sum(int(r[ix]) for r in data)
stot = sum(int(r[st]) for r in data)
print("total warp instr", tot, "samples", stot)
for i, r in enumerate(data):
    n = int(r[ix])
    if n > tot * thr or int(r[st]) > stot * 0.01:
        print(i, r[0][-5:], f"{n / tot * 100:5.2f}% ex {int(r[st]) / stot * 100:5.2f}% st thr{r[th]:>5}", r[1][:70])
