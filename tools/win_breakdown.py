"""One quarter-column window forward + adjoint of camera 1 (128^3 two-camera), for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_03358_b200 import lfm
from workloads import flame_volume, make_config, uniform_vector
cfg = make_config("128^3 two-camera")
plan = lfm.Plan(cfg, device=0)
ws = plan.workspace()
inf = plan.infos[1]
x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
y = torch.empty(inf["n_pix"], device="cuda:0")
r = torch.as_tensor(uniform_vector(inf["n_pix"], 1), device="cuda:0")
g = torch.empty_like(x)
for win in ((0, 2048, 0, 2048), (0, 2048, 1536, 2048)):
    lfm.A_forward_window(plan, 1, *win, x, y, ws)
    lfm.A_adjoint_window(plan, 1, *win, r, g, ws)
torch.cuda.synchronize()
