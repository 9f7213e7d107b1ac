"""Device time of the NEXT rows at the metric's scale (one JSON line): the A+A^T pair of the 128^3 hexagonal /
circular-aperture two-camera config (NEXT-4, T lenslet-stage terms) on the collapsed tcgen05 path and on the
per-view path, the cameras one after another on one stream, median of 20 pairs, L2 flushed (read) before each.

    python tools/next_timing.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import flame_volume, make_config, uniform_vector  # noqa: E402


def main():
    name = "128^3 hex two-camera"
    cfg = make_config(name)
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
    ys = [torch.empty(plan.infos[c]["n_pix"], device="cuda:0") for c in range(plan.n_cam)]
    rs = [torch.as_tensor(uniform_vector(plan.infos[c]["n_pix"], 1 + c), device="cuda:0") for c in range(plan.n_cam)]
    g = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, device="cuda:0")
    out = {"config": name, "s3_terms": [plan.infos[c]["s3_terms"] for c in range(plan.n_cam)]}
    for path, tag in ((lfm.COLLAPSED, "collapsed"), (lfm.PER_VIEW, "per_view")):
        def pair():
            for c in range(plan.n_cam):
                lfm.A_forward(plan, c, x, ys[c], ws, path=path)
            for c in range(plan.n_cam):
                lfm.A_adjoint(plan, c, rs[c], g, ws, accumulate=c > 0, path=path)
        for _ in range(3):
            pair()
        ts = []
        for _ in range(20 if path == lfm.COLLAPSED else 3):
            torch.sum(flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            pair()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        out[tag] = {"ms_per_pair": ms, "pairs_per_s": 1e3 / ms}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
