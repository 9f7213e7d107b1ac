import csv, sys, re
from collections import defaultdict
path, which = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
sections = []
cur = None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]; sections.append(cur); continue
    if r and r[0] == "Address":
        cur[1] = r; continue
    if cur and cur[1] and len(r) == len(cur[1]):
        cur[2].append(dict(zip(cur[1], r)))
sec = [s for s in sections if which in s[0]][0]
ins = sec[2]
tot_s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in ins)
tot_i = sum(int(d["Instructions Executed"] or 0) for d in ins)
op = defaultdict(lambda: [0, 0])
for d in ins:
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", d["Source"])
    o = m.group(2).split(".")[0] if m else "?"
    op[o][0] += int(d["Instructions Executed"] or 0); op[o][1] += int(d["Warp Stall Sampling (All Samples)"] or 0)
print(sec[0], "total warp-instr", tot_i, "samples", tot_s)
for o, (n, s) in sorted(op.items(), key=lambda x: -x[1][0])[:22]:
    print(f"{o:10s} {n:12d} {100*n/tot_i:5.1f}%  samples {100*s/max(tot_s,1):5.1f}%")
stall_cols = [c for c in sec[1] if c.startswith("stall_") and "Not Issued" not in c]
st = {c: sum(int(d[c] or 0) for d in ins) for c in stall_cols}
print("stalls:", sorted(((v, k) for k, v in st.items() if v), reverse=True)[:8])
