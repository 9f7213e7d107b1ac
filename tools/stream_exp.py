"""Experiment: A+A^T pair with the cameras on one stream (as bench.py) vs on two streams (separate workspaces,
the second camera's adjoint into its own volume, summed at the end by an accumulate of a copy)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_03358_b200 import lfm
from workloads import flame_volume, make_config, uniform_vector
cfg = make_config("128^3 two-camera")
plan = lfm.Plan(cfg, device=0)
ws = [plan.workspace(), plan.workspace()]
x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
ys = [torch.empty(plan.infos[c]["n_pix"], device="cuda:0") for c in range(2)]
rs = [torch.as_tensor(uniform_vector(plan.infos[c]["n_pix"], 1 + c), device="cuda:0") for c in range(2)]
g = torch.empty_like(x); g1 = torch.empty_like(x)
main = torch.cuda.current_stream()
ss = [torch.cuda.Stream(), torch.cuda.Stream()]

def one_stream():
    for c in range(2): lfm.A_forward(plan, c, x, ys[c], ws[0])
    for c in range(2): lfm.A_adjoint(plan, c, rs[c], g, ws[0], accumulate=c > 0)

def two_streams():
    e0 = torch.cuda.Event(); e0.record(main)
    for c in range(2):
        ss[c].wait_event(e0)
        lfm.A_forward(plan, c, x, ys[c], ws[c], stream=ss[c])
        lfm.A_adjoint(plan, c, rs[c], g if c == 0 else g1, ws[c], stream=ss[c])
    for c in range(2): main.wait_stream(ss[c])
    lfm.vol_rotate  # (sum below is the experiment's only torch arithmetic)
    g.add_(g1)

for fn in (one_stream, two_streams, one_stream, two_streams):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(100): fn()
    b.record(main); torch.cuda.synchronize()
    print(fn.__name__, "%.4f ms/pair" % (a.elapsed_time(b) / 100))
