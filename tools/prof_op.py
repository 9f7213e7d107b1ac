"""Run one operator of the hot path a few times (for ncu captures): python tools/prof_op.py fwd|adj collapsed|per_view CAM [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import flame_volume, make_config, uniform_vector  # noqa: E402

which, path, cam = sys.argv[1], sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = make_config(os.environ.get("LFM_CONFIG", "128^3 two-camera"))
plan = lfm.Plan(cfg, device=0)
ws = plan.workspace()
p = lfm.COLLAPSED if path == "collapsed" else lfm.PER_VIEW
x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
y = torch.as_tensor(uniform_vector(plan.infos[cam]["n_pix"], 1), device="cuda:0")
g = torch.empty_like(x)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
for i in range(reps):
    ev[2 * i].record()
    if which == "fwd":
        lfm.A_forward(plan, cam, x, y, ws, path=p)
    else:
        lfm.A_adjoint(plan, cam, y, g, ws, path=p)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
print(which, path, cam, ["%.3f ms" % ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps)])
