"""Per-source-line summary of an `ncu --page source --csv --print-source cuda,sass`
dump: warp-level instructions executed (split FP64 / other) and stall samples."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0  # e.g. warp-sweeps, to print per-unit counts
cur_file, cur_line, cur_src = "", None, ""
agg = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        cur_line, cur_src = r[0], r[1]
        continue
    sass = r[3].strip()
    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    n = f(r[7])
    s = f(r[4])
    op = sass.split()[1] if sass.startswith("@") else (sass.split()[0] if sass else "")
    key = (cur_file, cur_line)
    a = agg[key]
    a[3] = cur_src.strip()[:70]
    if op.startswith(("DFMA", "DMUL", "DADD", "DSETP")):
        a[0] += n
    else:
        a[1] += n
    a[2] += s
tot = sum(v[0] + v[1] for v in agg.values())
print(f"{'file:line':28s} {'fp64/u':>8s} {'other/u':>8s} {'samp%':>6s}  source")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][1]))[:45]:
    print(f"{k[0]+':'+k[1]:28s} {v[0]/norm:8.1f} {v[1]/norm:8.1f} {100*v[2]/max(1,sum(x[2] for x in agg.values())):6.2f}  {v[3]}")
