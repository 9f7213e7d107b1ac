"""One-line summary of a bench.py log: pairs/s and the per-kernel table times (us)."""
import json
import sys

for path in sys.argv[1:]:
    lines = [x for x in open(path) if x.startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    k = d.get("kernels", {})
    print(path, "pairs/s %.1f" % d["value"], {n: round(v["ms"] * 1e3, 1) for n, v in k.items()})
