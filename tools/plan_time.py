"""Time plan creation (host build + upload + autotune) for a config: python tools/plan_time.py [config]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "128^3 two-camera"
cfg = make_config(name)
t = time.time()
lfm.Plan(cfg, device=-1)
t_host = time.time() - t
t = time.time()
p = lfm.Plan(cfg, device=0)
t_dev = time.time() - t
print("%s: host build %.1f s, full plan (build + upload + autotune) %.1f s, tables %.0f MB" % (
    name, t_host, t_dev, sum(p.infos[c]["table_bytes"] for c in range(p.n_cam)) / 1e6))
