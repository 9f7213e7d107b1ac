"""Isolate a failing 2xFP16 launch: forward / adjoint of each camera of a config, synchronised after each call, errors
vs the fp64 oracle (small configs).  python tools/dbg_f16.py CONFIG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import make_config, uniform_vector, uniform_volume  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "small_two"
cfg = make_config(name)
plan = lfm.Plan(cfg, device=0)
ws = plan.workspace()
oracle = None
if cfg["volume"]["nx"] <= 32:
    from oracle.system import build_system
    oracle = build_system(cfg)
x = uniform_volume(cfg["volume"], 0)
for c in range(plan.n_cam):
    n_pix = plan.infos[c]["n_pix"]
    y = torch.empty(n_pix, device="cuda:0")
    lfm.A_forward(plan, c, torch.as_tensor(x, device="cuda:0").ravel(), y, ws)
    torch.cuda.synchronize()
    msg = "cam %d forward ok" % c
    if oracle:
        yr = oracle[c].forward(x.astype(np.float64))
        msg += " err %.3e" % (np.abs(y.cpu().numpy() - yr).max() / np.abs(yr).max())
    print(msg, flush=True)
    r = uniform_vector(n_pix, 1)
    g = torch.empty(plan.infos[c]["n_vox"], device="cuda:0")
    lfm.A_adjoint(plan, c, torch.as_tensor(r, device="cuda:0"), g, ws)
    torch.cuda.synchronize()
    msg = "cam %d adjoint ok" % c
    if oracle:
        gr = oracle[c].adjoint(r.astype(np.float64))
        msg += " err %.3e" % (np.abs(g.cpu().numpy() - gr).max() / np.abs(gr).max())
    print(msg, flush=True)
