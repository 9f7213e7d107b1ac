"""Angular-plane discretisation study (NEXT-3; paper sec,angular P:477-522): render the flame phantom with
the pillbox and Dirac angular bases at K = k x k views per camera and compare each rendering with the
highest-quality pinhole (Dirac) rendering by the normalised squared difference
    NSD(y) = ||a y - y_hq||^2 / ||y_hq||^2,
with a = <y, y_hq>/<y, y> the least-squares scale (reading R6: the paper's V normalisations leave the
absolute scale of y K-dependent (Z7), so the comparison is made up to one scalar; `nsd_raw` is the literal
formula).  Also times one forward projection per model on the per-view path (cost linear in K) and
on the K-collapsed path (cost independent of K).  All arithmetic runs in the CUDA library through the C ABI.

    python tools/angular_study.py [--config "64^3 single"] [--ks 1,2,4,8,16] [--ref 32] [--out results/...json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import flame_volume, make_config  # noqa: E402
from workloads.geometry import DIRAC, PILLBOX  # noqa: E402


def render(cfg, basis, k, x, reps=5):
    cam = dict(cfg["cameras"][0], basis=basis, k_s=k, k_t=k)
    c = dict(cfg, cameras=[cam])
    plan = lfm.Plan(c, device=0)
    ws = plan.workspace()
    y = torch.empty(plan.infos[0]["n_pix"], device="cuda:0")
    out = {}
    for path, name in [(lfm.PER_VIEW, "per_view"), (lfm.COLLAPSED, "collapsed")]:
        lfm.A_forward(plan, 0, x, y, ws, path=path)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            lfm.A_forward(plan, 0, x, y, ws, path=path)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[name + "_ms"] = sorted(ts)[len(ts) // 2]
    lfm.A_forward(plan, 0, x, y, ws, path=lfm.COLLAPSED)
    return y.double(), out


def nsd(y, ref):
    a = float((y * ref).sum() / (y * y).sum())
    d = float(((a * y - ref) ** 2).sum() / (ref ** 2).sum())
    raw = float(((y - ref) ** 2).sum() / (ref ** 2).sum())
    return d, raw, a


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="64^3 single")
    ap.add_argument("--ks", default="1,2,4,8,16")
    ap.add_argument("--ref", type=int, default=32)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = make_config(args.config)
    x = torch.as_tensor(flame_volume(cfg["volume"]), device="cuda:0").reshape(-1)
    t0 = time.time()
    ref, _ = render(cfg, DIRAC, args.ref, x, reps=1)
    rows = []
    for k in [int(v) for v in args.ks.split(",")]:
        for basis, bname in [(PILLBOX, "pillbox"), (DIRAC, "dirac")]:
            y, tm = render(cfg, basis, k, x)
            d, raw, a = nsd(y, ref)
            rows.append(dict(basis=bname, k=k, views=k * k, nsd=d, nsd_raw=raw, scale=a, **tm))
            print(json.dumps(rows[-1]))
    res = dict(config=args.config, reference="dirac %dx%d" % (args.ref, args.ref), rows=rows,
               seconds=time.time() - t0)
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
