"""One A_forward + A_adjoint of one camera between cudaProfilerStart/Stop (for `ncu --profile-from-start off`
captures of the whole per-camera chain):  python tools/prof_pair.py [CAM]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import flame_volume, make_config, uniform_vector  # noqa: E402

cam = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = make_config(os.environ.get("LFM_CONFIG", "128^3 two-camera"))
plan = lfm.Plan(cfg, device=0)
ws = plan.workspace()
x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
y = torch.empty(plan.infos[cam]["n_pix"], device="cuda:0")
r = torch.as_tensor(uniform_vector(plan.infos[cam]["n_pix"], 1), device="cuda:0")
g = torch.empty_like(x)
lfm.A_forward(plan, cam, x, y, ws)
lfm.A_adjoint(plan, cam, r, g, ws)
torch.cuda.synchronize()
torch.cuda.profiler.start()
lfm.A_forward(plan, cam, x, y, ws)
lfm.A_adjoint(plan, cam, r, g, ws)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
