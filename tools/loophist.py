"""Instruction histogram of an address range of a tools/sass.py -v dump."""
import collections
import sys

path, a, b = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
c = collections.Counter()
for line in open(path):
    if len(line) > 7 and line[6] == " ":
        try:
            ad = int(line[:6], 16)
        except ValueError:
            continue
        if a <= ad <= b:
            s = line[7:].split()
            op = s[1] if s[0].startswith("@") else s[0]
            c[op.split(".")[0]] += 1
fp64 = sum(v for k, v in c.items() if k in ("DFMA", "DMUL", "DADD", "DSETP"))
print(sum(c.values()), "instr, fp64", fp64, c.most_common(24))
