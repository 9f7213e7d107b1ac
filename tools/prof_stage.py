"""One stage kernel of the collapsed path between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures:  python tools/prof_stage.py fwd|adj [CAM] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import flame_volume, make_config, uniform_vector  # noqa: E402

which = sys.argv[1]
cam = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = make_config(os.environ.get("LFM_CONFIG", "128^3 two-camera"))
plan = lfm.Plan(cfg, device=0)
ws = plan.workspace()
x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
y = torch.empty(plan.infos[cam]["n_pix"], device="cuda:0")
r = torch.as_tensor(uniform_vector(plan.infos[cam]["n_pix"], 1), device="cuda:0")
lfm.A_forward(plan, cam, x, y, ws)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
torch.cuda.profiler.start()
for i in range(reps):
    torch.cuda._sleep(100000)  # keep the stream busy while the host enqueues (device time only)
    ev[2 * i].record()
    if which == "fwd":
        lfm.A_stage(plan, cam, lfm.STAGE_FWD_T, None, y, ws)
    else:
        lfm.A_stage(plan, cam, lfm.STAGE_ADJ_T, r, None, ws)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(which, cam, ["%.3f ms" % ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps)])
