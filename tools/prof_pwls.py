"""pwls_stats and the regulariser gradient (lfm_pwls_grad with no cameras) once each between cudaProfilerStart/Stop
at 256^3 (ncu --profile-from-start off captures):  python tools/prof_pwls.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import make_config, uniform_vector, uniform_volume  # noqa: E402

cfg = make_config(os.environ.get("LFM_CONFIG", "256^3 four-camera"))
plan = lfm.Plan(cfg, device=0)
ws = plan.workspace()
npx, nv = plan.infos[0]["n_pix"], plan.infos[0]["n_vox"]
x = torch.as_tensor(uniform_volume(cfg["volume"], 0), device="cuda:0").reshape(-1)
out = torch.empty_like(x)
y = torch.rand(npx, device="cuda:0")
r = torch.as_tensor(uniform_vector(npx, 1), device="cuda:0")
wts = torch.ones(npx, device="cuda:0")
stats = torch.zeros(3, dtype=torch.float64, device="cuda:0")
for _ in range(2):
    lfm.pwls_stats(plan, 0, y, r, wts, stats, ws)
    lfm.pwls_grad(plan, x, [], [], [], None, 0.01, 0.0, out, ws, cam0=0, cam1=0, include_reg=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
lfm.pwls_stats(plan, 0, y, r, wts, stats, ws)
lfm.pwls_grad(plan, x, [], [], [], None, 0.01, 0.0, out, ws, cam0=0, cam1=0, include_reg=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
