"""Per-kernel SASS dump and instruction histogram (cuobjdump), for quick checks here."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1]
pat = sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    if not re.search(pat, name):
        continue
    ins = []
    for line in f.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print("==", name, len(ins), "instructions")
    if "-v" in sys.argv:
        for a, s in ins:
            print(f"{a:06x} {s}")
    c = collections.Counter()
    for _, s in ins:
        op = s.split()[0]
        if op.startswith("@"):
            op = s.split()[1]
        c[op.split(".")[0]] += 1
    print(c.most_common(25))
