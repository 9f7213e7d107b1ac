#!/usr/bin/env python
"""Benchmark: A+A^T pairs/s of the plenoptic light-transport system model (arXiv 1812.03358).

One step = one pair: A_forward for every camera of the config, then A_adjoint for every camera
accumulated into one gradient volume (rotation passes included, plan build excluded) --
BASELINE.json's metric on its 128^3 two-camera config (configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--path collapsed|per_view]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: cameras x detector-row tiles)

Timing: W untimed steps, then K steps; between steps L2 is flushed (a 256 MiB write); each step is
bracketed by CUDA events on the launching stream (the flush is outside the events); the whole loop is
bracketed by a barrier + synchronize; rank 0 prints ONE JSON line with the max over ranks.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "128^3 two-camera"
METRIC = "A+A^T pairs/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="collapsed", choices=["collapsed", "per_view"])
    ap.add_argument("--config", default=WORKLOAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-per-view", action="store_true", help="skip the per-view path reference timing")
    ap.add_argument("--one-stream", action="store_true", help="run the rank's cameras one after another on one stream")
    ap.add_argument("--no-graph", action="store_true", help="launch the timed pairs eagerly instead of as a CUDA graph")
    return ap.parse_args()


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [v.strip() for v in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------ helpers
def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic():
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
    except Exception:
        return {}


def cpu_baseline(cfg, n_views_sample=None):
    """Oracle (fp64, as it stands) timed on this host: camera 0 forward + adjoint on a view sample,
    scaled linearly in K and by the number of cameras; rotation timed separately."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle.camera import CameraModel
    from oracle.rotation import Rotation
    from workloads import flame_volume, uniform_vector
    vol = cfg["volume"]
    dims = (vol["nx"], vol["ny"], vol["nz"])
    vox = (vol["dx"], vol["dy"], vol["dz"])
    with threadpool_limits(limits=1):
        cam = CameraModel(cfg["cameras"][0], dims, vox)
        K = cam.ks * cam.kt
        views = [(ks, kt) for kt in range(cam.kt) for ks in range(cam.ks)]
        if n_views_sample:
            views = views[:n_views_sample]
        x = flame_volume(vol).astype(np.float64)
        r = uniform_vector(cam.n_pix, 1).astype(np.float64)
        t0 = time.perf_counter()
        cam.forward(x, views=views)
        cam.adjoint(r, views=views)
        t_cam = (time.perf_counter() - t0) * K / len(views)
        t_rot = 0.0
        for c in cfg["cameras"][1:]:
            rot = Rotation(c["R"], dims, vox)
            t0 = time.perf_counter()
            rot.adjoint(rot.forward(x))
            t_rot += time.perf_counter() - t0
    t_pair = t_cam * len(cfg["cameras"]) + t_rot
    return dict(value=1.0 / t_pair, unit="pairs/s", cores=1, kind="oracle",
                sample="camera 0 fwd+adj over %d of %d views, scaled x%d views and x%d cameras, + measured "
                       "rotation fwd+adj of the posed cameras; single thread (scipy.sparse fp64)"
                       % (len(views), K, K // len(views), len(cfg["cameras"])),
                seconds_measured=round(t_cam * len(views) / K + t_rot, 2))


# ------------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The oracle as the reference arm (tier rule): bounded samples of the same workload on host cores."""
    if rank != 0:
        return
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle.system import SystemOperator
    from workloads import flame_volume, make_config, uniform_vector
    cfg = make_config(args.config)
    t_build = time.perf_counter()
    ops = [SystemOperator(cfg["volume"], c) for c in cfg["cameras"]]
    t_build = time.perf_counter() - t_build
    x = flame_volume(cfg["volume"]).astype(np.float64)
    rs = [uniform_vector(op.n_pix, 1).astype(np.float64) for op in ops]
    K = ops[0].camera.ks * ops[0].camera.kt
    per_view, per_rot = [], []
    with threadpool_limits(limits=1):
        for it in range(args.warmup + args.steps):
            k = it % K
            view = [(k % ops[0].camera.ks, k // ops[0].camera.ks)]
            t_rot = 0.0
            t_cam = 0.0
            for op, r in zip(ops, rs):
                t0 = time.perf_counter()
                xr = op.rot.forward(x)
                t1 = time.perf_counter()
                op.camera.forward(xr, views=view)
                gr = op.camera.adjoint(r, views=view)
                t2 = time.perf_counter()
                op.rot.adjoint(gr)
                t3 = time.perf_counter()
                t_rot += (t1 - t0) + (t3 - t2)
                t_cam += t2 - t1
            if it >= args.warmup:
                per_view.append(t_cam)
                per_rot.append(t_rot)
    # one step = one view of every camera's forward+adjoint (+ the rotations, once per pair); a full pair
    # is K views (cost linear in K)
    t_pair = (sum(per_view) / len(per_view)) * K + sum(per_rot) / len(per_rot)
    value = 1.0 / t_pair
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_pair, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "step": "one view of an A+A^T pair per timed step, x%d views" % K},
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": 1, "kind": "oracle",
                             "sample": "per step: 1 of %d views of every camera's fwd+adj with rotation; "
                                       "oracle build %.1fs excluded" % (K, t_build)},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1812_03358_b200 import lfm
    from paper_1812_03358_b200.parallel import ConcurrentPair, PairRunner, shard
    from workloads import flame_volume, make_config, uniform_vector
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = make_config(args.config)
    path = lfm.COLLAPSED if args.path == "collapsed" else lfm.PER_VIEW
    plan = lfm.Plan(cfg, device=local_rank)
    ws = plan.workspace()
    items = shard([c["n_t"] for c in cfg["cameras"]], rank, world)
    n_vox = plan.infos[0]["n_vox"]
    x = torch.as_tensor(flame_volume(cfg["volume"]), device=dev).reshape(-1)
    ys = {c: torch.empty(plan.infos[c]["n_pix"], device=dev) for c, _, _ in items}
    rs = {c: torch.as_tensor(uniform_vector(plan.infos[c]["n_pix"], 1 + c), device=dev) for c, _, _ in items}
    g = torch.empty(n_vox, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    launches = [0]

    def fwd_rows(c, r0, r1, xv, y):
        lfm.A_forward_rows(plan, c, r0, r1, xv, y, ws, path=path)
        launches[0] += lfm.last_launch_count()

    def adj_rows(c, r0, r1, r, gv, acc):
        lfm.A_adjoint_rows(plan, c, r0, r1, r, gv, ws, accumulate=acc, path=path)
        launches[0] += lfm.last_launch_count()

    def allreduce(gv):
        dist.all_reduce(gv)
        launches[0] += 1

    if len(items) > 1 and not args.one_stream:
        # the rank's items (cameras / row tiles) run concurrently, each on its own stream and workspace; the
        # backprojections of items >= 1 go to private volumes added into g in item order (ConcurrentPair)
        streams = [torch.cuda.Stream(device=dev) for _ in items]
        wss = [ws] + [plan.workspace() for _ in items[1:]]
        private = [None] + [torch.empty(n_vox, device=dev) for _ in items[1:]]
        start = torch.cuda.Event()

        def run(i, fn):
            s_i = streams[i]
            s_i.wait_event(start)
            with torch.cuda.stream(s_i):
                fn()

        def join():
            cur = torch.cuda.current_stream()
            for s_i in streams:
                cur.wait_stream(s_i)

        def accumulate(src, dst):
            lfm.vol_accumulate(src, dst)
            launches[0] += lfm.last_launch_count()

        def fwd_i(i, c, r0, r1, xv, y):
            lfm.A_forward_rows(plan, c, r0, r1, xv, y, wss[i], path=path)
            launches[0] += lfm.last_launch_count()

        def adj_i(i, c, r0, r1, r, gv):
            lfm.A_adjoint_rows(plan, c, r0, r1, r, gv, wss[i], accumulate=False, path=path)
            launches[0] += lfm.last_launch_count()

        runner = ConcurrentPair(items, fwd_i, adj_i, accumulate, lambda gv: gv.zero_(), run, join, private,
                                allreduce if world > 1 else None)
    else:
        start = None
        runner = PairRunner(items, fwd_rows, adj_rows, lambda gv: gv.zero_(), allreduce if world > 1 else None)

    def step(x_in, g_out):
        launches[0] = 0
        if start is not None:
            start.record(torch.cuda.current_stream())
        runner.pair(x_in, ys, rs, g_out)

    # dominant kernel: the separable transport of an unrotated camera (one sep_kernel launch per call)
    dom_cam = next((c for c, r0, r1 in items if plan.infos[c]["rot_passes"] == 0 and r0 == 0
                    and r1 == plan.infos[c]["n_t"]), None)

    for _ in range(args.warmup):
        step(x, g)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the timed pair as one CUDA graph (captured once after the warm-up: the same kernels, tensor maps and
    # stream fork/join, replayed without host launch overhead); --no-graph launches it eagerly every step
    graph = None
    if not args.no_graph and world == 1:  # multi-rank pairs hold an NCCL all-reduce: launched eagerly
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step(x, g)
        n_graph_launches = launches[0]
        graph.replay()
        torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        if graph is not None:
            graph.replay()
        else:
            step(x, g)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    ms_mean = sum(ms) / len(ms)
    # dominant-kernel timing on the same stream, inside timed steps of the same shape
    # The dominant kernel of the collapsed path is its forward t pass (one launch, lfm_A_stage FWD_T:
    # the slice sum over the interleaved intermediate); its adjoint counterpart is ADJ_T.  Each launch
    # is timed alone with events on the bench stream, after an L2 flush, inputs from a full call.
    dom = None
    if dom_cam is not None:
        fwd_ms, adj_ms = [], []
        staged = path == lfm.COLLAPSED
        for i in range(max(3, args.steps // 2)):
            a, b, c_, d = (torch.cuda.Event(enable_timing=True) for _ in range(4))
            if staged:
                try:
                    lfm.A_forward(plan, dom_cam, x, ys[dom_cam], ws, path=path)
                    flush.zero_()
                    a.record(stream)
                    lfm.A_stage(plan, dom_cam, lfm.STAGE_FWD_T, None, ys[dom_cam], ws)
                    b.record(stream)
                    flush.zero_()
                    c_.record(stream)
                    lfm.A_stage(plan, dom_cam, lfm.STAGE_ADJ_T, rs[dom_cam], None, ws)
                    d.record(stream)
                except lfm.LfmError:  # fused collapsed forward: time the whole call instead
                    staged = False
            if not staged:
                flush.zero_()
                a.record(stream)
                lfm.A_forward(plan, dom_cam, x, ys[dom_cam], ws, path=path)
                b.record(stream)
                flush.zero_()
                c_.record(stream)
                lfm.A_adjoint(plan, dom_cam, rs[dom_cam], g, ws, path=path)
                d.record(stream)
            torch.cuda.synchronize()
            fwd_ms.append(a.elapsed_time(b))
            adj_ms.append(c_.elapsed_time(d))
        inf = plan.infos[dom_cam]
        kind = None
        if staged:
            fma_f, fma_a = inf["fma_stage"][0], inf["fma_stage"][1]
            kind = inf["kind_stage"][0]
            kname = "collapsed forward t pass (lfm_A_stage FWD_T), camera %d" % dom_cam
        else:
            fma_f = fma_a = inf["fma_alg"][1 if path == lfm.COLLAPSED else 0]
            kname = "%s A_forward, camera %d" % (args.path, dom_cam)
        dom = dict(fwd_ms=sum(fwd_ms) / len(fwd_ms), adj_ms=sum(adj_ms) / len(adj_ms), fma=fma_f, fma_adj=fma_a,
                   name=kname, kind=kind, mma=inf["mma_stage"][0])
    # the paper's own evaluation order (per-view factored chain) on the same
    # workload, for reference: device time of one forward and one adjoint per camera
    per_view = None
    if world == 1 and path == lfm.COLLAPSED and not args.no_per_view:
        fv, av = [], []
        for c in range(plan.n_cam):
            lfm.A_forward(plan, c, x, ys[c], ws, path=lfm.PER_VIEW)
            tf, ta = [], []
            for _ in range(3):
                a_, b_, c_, d_ = (torch.cuda.Event(enable_timing=True) for _ in range(4))
                flush.zero_()
                a_.record(stream)
                lfm.A_forward(plan, c, x, ys[c], ws, path=lfm.PER_VIEW)
                b_.record(stream)
                flush.zero_()
                c_.record(stream)
                lfm.A_adjoint(plan, c, rs[c], g, ws, path=lfm.PER_VIEW)
                d_.record(stream)
                torch.cuda.synchronize()
                tf.append(a_.elapsed_time(b_))
                ta.append(c_.elapsed_time(d_))
            fv.append(sorted(tf)[1])
            av.append(sorted(ta)[1])
        per_view = {"fwd_ms": fv, "adj_ms": av, "pairs_per_s": 1e3 / (sum(fv) + sum(av))}
    sm = clocks.stop()
    # e2e: through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        # Each step copies its own input volume host->device and its gradient device->host (pinned buffers,
        # two of each so step i+1's upload and step i's download overlap step i's / i+1's compute on a
        # separate copy stream; events order the buffers).
        xh = [x.cpu().pin_memory(), x.cpu().pin_memory()]
        gh = [torch.empty(n_vox, dtype=torch.float32).pin_memory() for _ in range(2)]
        xd = [torch.empty_like(x), torch.empty_like(x)]
        gd = [torch.empty_like(g), torch.empty_like(g)]
        cs = torch.cuda.Stream()

        def run_e2e(n):
            up = [torch.cuda.Event() for _ in range(n + 1)]
            done = [torch.cuda.Event() for _ in range(n)]
            cs.wait_stream(stream)  # nothing on the copy stream starts before the timed region opens
            with torch.cuda.stream(cs):
                xd[0].copy_(xh[0], non_blocking=True)
                up[0].record(cs)
            for i in range(n):
                stream.wait_event(up[i])
                step(xd[i % 2], gd[i % 2])
                done[i].record(stream)
                with torch.cuda.stream(cs):
                    if i + 1 < n:
                        if i >= 1:
                            cs.wait_event(done[i - 1])  # xd[(i+1)%2] was step i-1's input
                        xd[(i + 1) % 2].copy_(xh[(i + 1) % 2], non_blocking=True)
                        up[i + 1].record(cs)
                    cs.wait_event(done[i])
                    gh[i % 2].copy_(gd[i % 2], non_blocking=True)
            stream.wait_stream(cs)

        run_e2e(3)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_e2e(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / args.steps
        e2e = dict(ms=e2e_ms, h2d=xh[0].numel() * 4, d2h=gh[0].numel() * 4)
    # max over ranks
    t = torch.tensor([ms_mean, e2e["ms"] if e2e else 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_mean, e2e_ms = float(t[0]), float(t[1])
    if rank != 0:
        return
    peaks = measured_peaks()
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    fp32_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12   # TFLOP/s, DESIGN.md §roofline
    roof = None
    if dom is not None:
        achieved = 2.0 * dom["fma"] / (dom["fwd_ms"] * 1e-3) / 1e12
        tr = ncu_traffic().get("dominant_kernel_dram_bytes_per_launch")
        roof = {"bound": "alu", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": achieved / fp32_peak, "traffic": tr,
                "kernel": dom["name"],
                "kernel_ms": dom["fwd_ms"], "adjoint_kernel_ms": dom["adj_ms"],
                "adjoint_achieved": 2.0 * dom["fma_adj"] / (dom["adj_ms"] * 1e-3) / 1e12,
                "peak_note": "FP32 FMA: 148 SM x 128 lanes x 2 flop x %.0f MHz (sm_max_mhz, MEASURED_PEAKS.json)"
                             % sm_max}
        if dom.get("kind") == 8:
            # the stage runs on the tcgen05 tensor cores (band_u, 3xTF32): its roof is the tf32 tensor peak =
            # measured bf16 peak x nominal tf32/bf16 ratio (1.1 / 2.25, B200_PROFILING.md).  `achieved` stays the
            # algorithmic (non-zero) work; `issued` is the dense 3xTF32 MMA work the kernel actually runs
            # (block density x 3 products above the algorithm), `alu_equiv` the same time against the FP32 roof.
            tf32_peak = peaks.get("bf16_tflops", 1653.4) * 1.1 / 2.25
            issued = 2.0 * dom["mma"] / (dom["fwd_ms"] * 1e-3) / 1e12
            roof.update({"bound": "tensor", "peak": tf32_peak, "frac": achieved / tf32_peak,
                         "peak_note": "tf32 dense tensor peak = MEASURED_PEAKS bf16_tflops %.1f x 1.1/2.25 (nominal "
                                      "tf32/bf16 ratio, B200_PROFILING.md)" % peaks.get("bf16_tflops", 1653.4),
                         "issued": {"achieved": issued, "frac": issued / tf32_peak,
                                    "what": "3xTF32 dense 128x16-block MACs x 2 per launch / time"},
                         "alu_equiv": {"peak": fp32_peak, "frac": achieved / fp32_peak,
                                       "what": "algorithmic flops / time vs the FP32 FMA roof the plain kernels face"},
                         "kernel": dom["name"] + " on tcgen05 (band_u)"})
    pair_bytes = sum(plan.infos[c]["bytes_alg"][1 if path == lfm.COLLAPSED else 0] * 2 for c in range(plan.n_cam))
    value = 1e3 / ms_mean
    line = {"metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_mean, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "volume": "%d^3 flame phantom" % cfg["volume"]["nx"],
                       "cameras": len(cfg["cameras"]), "detector": "%dx%d" % (cfg["cameras"][0]["n_s"],
                                                                                cfg["cameras"][0]["n_t"]),
                       "views": "%dx%d pillbox" % (cfg["cameras"][0]["k_s"], cfg["cameras"][0]["k_t"]),
                       "path": args.path, "parallelism": "cameras x detector-row tiles over %d rank(s)%s" % (
                           world, ", concurrent per-camera streams" if len(items) > 1 and not args.one_stream else ""),
                       "l2": "256 MiB write between steps, outside the per-step CUDA events",
                       "launch": "eager" if (args.no_graph or world > 1) else "one CUDA graph per pair (captured after warm-up)"},
            "hbm_gbs_alg": pair_bytes / (ms_mean * 1e-3) / 1e9,
            "hbm_frac_of_measured": pair_bytes / (ms_mean * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6551.4),
            "roofline": roof, "clocks": sm, "gpu_launches": launches[0] * args.steps}
    if per_view is not None:
        line["per_view_path"] = per_view
    if e2e:
        line["e2e"] = {"value": 1e3 / e2e_ms, "unit": "pairs/s", "h2d_bytes_per_step": e2e["h2d"],
                       "d2h_bytes_per_step": e2e["d2h"]}
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg)
        except Exception as exc:  # the baseline is a report, never a reason to lose the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "pairs/s", "cores": 1, "kind": "oracle",
                                    "sample": "failed: %s" % exc}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
