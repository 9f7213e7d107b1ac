"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0, ""])
line = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        line = (r[0], r[1][:90])
    try:
        n = int(r[7] or 0)
        s = int(r[4] or 0)
    except ValueError:
        continue
    agg[line][0] += n
    agg[line][1] += s
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*v[0]/tot:5.1f}% instr {100*v[1]/tots:5.1f}% samples  L{k[0]}: {k[1]}")
