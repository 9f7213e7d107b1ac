"""HBM-bound kernels of the pair and of the PWLS step timed alone at a volume size where launch overhead does
not dominate: the 256^3 four-camera config (BASELINE configs[3], 64 MiB volumes, 2048^2 detectors), camera 0
(yaw -30: z and x shear passes) and camera 3 (pitch +30: z and y passes).  Median of 15 launches, L2 flushed
before each by reading a 256 MiB buffer; algorithmic bytes as in bench.py's kernel table.  One JSON line.

    python tools/hbm_kernels.py [config]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402
from workloads import make_config, uniform_vector, uniform_volume  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "256^3 four-camera"
    cfg = make_config(name)
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) \
        if os.path.exists("MEASURED_PEAKS.json") else {}
    hbm = peaks.get("hbm_gbs", 6550.1)
    nv = plan.infos[0]["n_vox"]
    npx = plan.infos[0]["n_pix"]
    x = torch.as_tensor(uniform_volume(cfg["volume"], 0), device="cuda:0").reshape(-1)
    out = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, device="cuda:0")

    def timed(fn, reps=15):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            torch.sum(flush)
            torch.cuda._sleep(100000)  # the stream stays busy while the host enqueues fn (device time only)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return sorted(ts)[len(ts) // 2]

    res = {"config": name, "hbm_peak_gbs": hbm, "flush": "256 MiB read before each launch", "kernels": {}}

    def add(k, ms, nbytes, what):
        gbs = nbytes / (ms * 1e-3) / 1e9
        res["kernels"][k] = {"us": round(ms * 1e3, 2), "bytes": nbytes, "gbs": round(gbs, 1),
                             "frac_measured": round(gbs / hbm, 3), "frac_8tbs": round(gbs / 8000, 3), "what": what}

    for c in range(plan.n_cam):
        passes = bin(plan.infos[c]["rot_passes"] & 7).count("1")
        if passes and c in (0, 3):
            add("rotation_fwd cam%d" % c, timed(lambda: lfm.vol_rotate(plan, c, lfm.FWD, x, out, ws)), 8.0 * nv * passes,
                "%d shear passes, read + write per voxel per pass" % passes)
            add("rotation_adj cam%d" % c, timed(lambda: lfm.vol_rotate(plan, c, lfm.ADJ, x, out, ws)), 8.0 * nv * passes,
                "%d shear passes" % passes)
    inf = plan.infos[1]
    z_bytes = 4.0 * inf["ny"] * inf["nz"] * inf["n_s"]
    y = torch.empty(npx, device="cuda:0")
    r = torch.as_tensor(uniform_vector(npx, 1), device="cuda:0")
    add("s_pass_fwd (band_v)", timed(lambda: lfm.A_stage(plan, 1, lfm.STAGE_FWD_S, x, None, ws)), 4.0 * nv + z_bytes,
        "read x^r, write U")
    lfm.A_stage(plan, 1, lfm.STAGE_ADJ_T, r, None, ws)
    add("s_pass_adj (band_v)", timed(lambda: lfm.A_stage(plan, 1, lfm.STAGE_ADJ_S, None, out, ws)), z_bytes + 4.0 * nv,
        "read Z, write x^r")
    stats = torch.zeros(3, dtype=torch.float64, device="cuda:0")
    wts = torch.ones(npx, device="cuda:0")
    add("pwls_stats", timed(lambda: lfm.pwls_stats(plan, 1, y, r, wts, stats, ws)), 12.0 * npx, "read Ax, y, w")
    add("pwls_reg26 (+fill)", timed(lambda: lfm.pwls_grad(plan, x, [], [], [], None, 0.01, 0.0, out, ws, cam0=0, cam1=0,
                                                          include_reg=True)), 16.0 * nv, "write grad, read x, read+write grad")
    zz, dd, gg = torch.rand(nv, device="cuda:0"), torch.rand(nv, device="cuda:0") + 1.0, torch.rand(nv, device="cuda:0")
    xx = torch.rand(nv, device="cuda:0")
    add("fista_update", timed(lambda: lfm.fista_update(plan, xx, zz, gg, dd, 1.0, 1.6)), 24.0 * nv,
        "read x, z, grad, d; write x, z")
    add("vol_accumulate", timed(lambda: lfm.vol_accumulate(gg, out)), 12.0 * nv, "dst += src")
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
