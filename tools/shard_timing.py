"""Per-rank device time of the multi-GPU shards: A_forward_window / A_adjoint_window of one
camera of the 128^3 two-camera config on 1, 2, 4 and 8 column tiles (the default partition) and row tiles,
median of 20 launches each after an L2 flush, on one GPU.  The largest tile of each split is timed (the rank
that bounds the step).  Prints one JSON line; the 8-GPU prediction of DESIGN.md §7 is computed from it.

    python tools/shard_timing.py [camera]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from paper_1812_03358_b200.parallel import _split  # noqa: E402
from workloads import flame_volume, make_config, uniform_vector  # noqa: E402


def main():
    cam = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cfg = make_config("128^3 two-camera")
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    inf = plan.infos[cam]
    n_t, n_s = inf["n_t"], inf["n_s"]
    x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
    y = torch.empty(inf["n_pix"], device="cuda:0")
    r = torch.as_tensor(uniform_vector(inf["n_pix"], 1), device="cuda:0")
    g = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, device="cuda:0")

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        out = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b))
        return sorted(out)[len(out) // 2]

    res = {"camera": cam, "config": "128^3 two-camera", "pose": list(cfg["cameras"][cam]["R"])}
    for axis in ("cols", "rows"):
        for tiles in (1, 2, 4, 8):
            parts = _split(n_s if axis == "cols" else n_t, tiles, 256 if axis == "cols" else 1)
            best = None
            for a0, a1 in parts:
                win = (0, n_t, a0, a1) if axis == "cols" else (a0, a1, 0, n_s)
                f = timed(lambda: lfm.A_forward_window(plan, cam, *win, x, y, ws))
                d = timed(lambda: lfm.A_adjoint_window(plan, cam, *win, r, g, ws))
                if best is None or f + d > best[0] + best[1]:
                    best = (f, d, win)
            res["%s_1/%d" % (axis, tiles)] = {"fwd_ms": best[0], "adj_ms": best[1], "window": best[2]}
    full = res["cols_1/1"]
    for k, v in res.items():
        if isinstance(v, dict) and "fwd_ms" in v:
            v["fwd_frac"] = v["fwd_ms"] / full["fwd_ms"]
            v["adj_frac"] = v["adj_ms"] / full["adj_ms"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
