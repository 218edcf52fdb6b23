"""Summarise an `ncu --page source --csv --print-source sass` dump: samples and
executed instructions per opcode, and the hottest instructions."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
col = {k: h.index(k) for k in h}
data = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
S, I, T = col["Warp Stall Sampling (All Samples)"], col["Instructions Executed"], col["Thread Instructions Executed"]
stall_cols = [k for k in h if k.startswith("stall_")]
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
by_op = defaultdict(lambda: [0.0, 0.0, 0.0])
tot_s = sum(num(r[S]) for r in data)
for r in data:
    op = r[col["Source"]].split()[0] if r[col["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[col["Source"]].split()[1]
    op = op.split(".")[0]
    by_op[op][0] += num(r[S]); by_op[op][1] += num(r[I]); by_op[op][2] += num(r[T])
tot_i = sum(v[1] for v in by_op.values())
print(f"total samples {tot_s:.0f}, warp-instr {tot_i:.3e}")
print(f"{'op':10s} {'samples%':>8s} {'instr%':>7s} {'thr/inst':>8s}")
for op, (s, i, t) in sorted(by_op.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{op:10s} {100*s/tot_s:8.2f} {100*i/tot_i:7.2f} {t/max(i,1):8.2f}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("\nhottest instructions:")
for r in sorted(data, key=lambda r: -num(r[S]))[:n]:
    st = sorted(((num(r[col[k]]), k[6:]) for k in stall_cols), reverse=True)[:3]
    print(f"{r[col['Address']]:>6s} {num(r[S]):7.0f} thr={num(r[T])/max(num(r[I]),1):5.1f} {r[col['Source']][:60]:60s} {st}")
