"""Summarise an `ncu --set full --page raw --csv` capture of one cfg2 multiply
(tools/profile_step.py --reps 1) into profiles/ncu_traffic.json: DRAM bytes
read + written by the numeric-phase kernels (k_push* / k_pull*), per multiply
— the `roofline.traffic` field of bench.py."""
import csv, json, sys

src, out = sys.argv[1], sys.argv[2]
lines = open(src).read().splitlines()
lines = lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):]   # drop ncu's preamble
rows = list(csv.reader(lines))
hdr = rows[0]
units = rows[1]
col = {k: i for i, k in enumerate(hdr)}


def val(r, name):
    v = r[col[name]].replace(",", "")
    u = units[col[name]]
    x = float(v)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
             "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(u, 1)
    return x * scale


kern = []
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if "k_push" not in name and "k_pull" not in name:
        continue
    kern.append({"kernel": name[:60],
                 "dram_read_bytes": val(r, "dram__bytes_read.sum"),
                 "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                 "l2_read_bytes_from_sm": val(r, "lts__t_sectors_srcunit_tex_op_read.sum") * 32,
                 "ncu_ms": val(r, "gpu__time_duration.sum")})
rd = sum(k["dram_read_bytes"] for k in kern)
wr = sum(k["dram_write_bytes"] for k in kern)
import subprocess
try:
    commit = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip()
except Exception:
    commit = None
json.dump({"source": "ncu --set full --clock-control none capture of one cfg2 multiply "
                     "(tools/profile_step.py --reps 1, algorithm=auto), numeric-phase kernels k_push*/k_pull*",
           "commit": sys.argv[3] if len(sys.argv) > 3 else commit,
           "config": "cfg2: R-MAT s20 ef16, L = tril(relabel(G)), C = L.(L L) plus-pair int64, auto",
           "command": "ncu --set full --clock-control none -k regex:'k_push|k_pull' --csv --page raw "
                      "python tools/profile_step.py --reps 1",
           "numeric_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
           "ncu_ms_sum": sum(k["ncu_ms"] for k in kern), "kernels": kern},
          open(out, "w"), indent=1)
print("numeric DRAM bytes", rd + wr, "kernels", len(kern))
