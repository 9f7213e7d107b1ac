"""Device time of A_forward_rows / A_adjoint_rows for 1, 2 and 4 row tiles of camera 0 (the per-rank work of the
multi-GPU partition), 128^3 two-camera config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_03358_b200 import lfm
from workloads import flame_volume, make_config, uniform_vector
cfg = make_config("128^3 two-camera")
plan = lfm.Plan(cfg, device=0)
ws = plan.workspace()
x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
nt = plan.infos[0]["n_t"]
y = torch.empty(plan.infos[0]["n_pix"], device="cuda:0")
r = torch.as_tensor(uniform_vector(plan.infos[0]["n_pix"], 1), device="cuda:0")
g = torch.empty_like(x)
for tiles in (1, 2, 4):
    r0, r1 = 0, nt // tiles
    for fn, name in ((lambda: lfm.A_forward_rows(plan, 0, r0, r1, x, y, ws), "fwd"),
                     (lambda: lfm.A_adjoint_rows(plan, 0, r0, r1, r, g, ws), "adj")):
        for _ in range(3): fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): fn()
        b.record(); torch.cuda.synchronize()
        print("rows 1/%d %s %.4f ms" % (tiles, name, a.elapsed_time(b) / 20))
