"""Per-launch table of an ncu --csv launch list with gpu__time_duration and DRAM bytes: one row per launch in order,
then the per-kernel totals.  python tools/launch_seq.py launches.csv [N_ROWS]"""
import csv
import sys
from collections import OrderedDict, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
nmax = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
cur = OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        cur.setdefault((d["ID"], d["Kernel Name"][:48]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, ((lid, k), d) in enumerate(cur.items()):
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    b = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    if i < nmax:
        print(f"{lid:>4} {k:50s} {t:7.1f} us {b:7.1f} MB {b / t / 1e3 if t else 0:5.2f} TB/s")
    agg[k][0] += 1
    agg[k][1] += t
    agg[k][2] += b
tot = sum(v[1] for v in agg.values())
print("--- totals")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:4d} {k:50s} {t:8.1f} us {100 * t / tot:5.1f}%  avg {t / n:6.1f} us  {b / t / 1e3:5.2f} TB/s")
