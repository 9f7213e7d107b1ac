"""Warm device time of the pieces of one camera's A_forward / A_adjoint (128^3 two-camera, camera 1 = posed):
rotation (vol_rotate fwd/adj), the whole forward / adjoint, and the t-pass stages."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_03358_b200 import lfm
from workloads import flame_volume, make_config, uniform_vector
cfg = make_config("128^3 two-camera")
plan = lfm.Plan(cfg, device=0)
ws = plan.workspace()
x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
xr = torch.empty_like(x); g = torch.empty_like(x)
def t(fn, n=50):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
for c in range(2):
    y = torch.empty(plan.infos[c]["n_pix"], device="cuda:0")
    r = torch.as_tensor(uniform_vector(plan.infos[c]["n_pix"], 1), device="cuda:0")
    print("cam", c, "rot_passes", plan.infos[c]["rot_passes"])
    print("  A_forward %.1f us" % t(lambda: lfm.A_forward(plan, c, x, y, ws)))
    print("  A_adjoint %.1f us" % t(lambda: lfm.A_adjoint(plan, c, r, g, ws)))
    print("  t pass fwd %.1f us" % t(lambda: lfm.A_stage(plan, c, lfm.STAGE_FWD_T, None, y, ws)))
    print("  t pass adj %.1f us" % t(lambda: lfm.A_stage(plan, c, lfm.STAGE_ADJ_T, r, None, ws)))
    if plan.infos[c]["rot_passes"]:
        print("  rotate fwd %.1f us" % t(lambda: lfm.vol_rotate(plan, c, 0, x, xr, ws)))
        print("  rotate adj %.1f us" % t(lambda: lfm.vol_rotate(plan, c, 1, x, xr, ws)))
