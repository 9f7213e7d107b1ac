"""Summarise ncu captures into profiles/: per-kernel raw metrics and the launch-list shares.

    python tools/summarize_profiles.py ROUND launches.csv prof1.ncu-rep [prof2.ncu-rep ...]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fma.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for w in WANT:
            if w in h:
                d[w] = (r[h.index(w)], units[h.index(w)])
        res.append(d)
    return res


def to_bytes(v):
    val, unit = v
    val = float(val.replace(",", ""))
    return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    rnd, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    pdir = os.path.join(ROOT, "profiles")
    os.makedirs(pdir, exist_ok=True)
    lines = []
    rows = list(csv.reader(open(launches)))
    hdr, agg = None, defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"][:90]][0] += 1
                agg[d["Kernel Name"][:90]][1] += float(d["Metric Value"].replace(",", ""))
    ours = {k: v for k, v in agg.items() if "lfm::" in k}
    tot = sum(v[1] for v in ours.values())
    cmd = os.environ.get("LAUNCH_CMD", "python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e")
    lines.append("# launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised:")
    lines.append(f"# compare shares, not absolutes) of `{cmd}`")
    lines.append("# share = of the lfm:: kernels' total; other launches (torch fills / reductions: the L2 flush between")
    lines.append("# steps, input init) are listed after, without a share")
    for k, (n, t) in sorted(ours.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n:4d} launches {t / 1e3:10.1f} us {100 * t / tot:5.1f}%  {k}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if k not in ours:
            lines.append(f"{n:4d} launches {t / 1e3:10.1f} us     -   {k}")
    open(os.path.join(pdir, f"{rnd}_launches.txt"), "w").write("\n".join(lines) + "\n")
    summary = {}
    for rep in reps:
        name = os.path.splitext(os.path.basename(rep))[0]
        res = [d for d in raw(rep) if "lfm::" in d["kernel"] or "band_" in d["kernel"]]  # not the spin / flush kernels
        txt = [f"# ncu --set full --clock-control none capture: {os.path.basename(rep)}"]
        for d in res:
            txt.append(d["kernel"])
            for k, v in d.items():
                if k != "kernel":
                    txt.append(f"  {k:70s} {v[0]:>18s} {v[1]}")
        open(os.path.join(pdir, f"{rnd}_{name}.txt"), "w").write("\n".join(txt) + "\n")
        summary[name] = [{"kernel": d["kernel"],
                          "dram_bytes": to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"]),
                          "duration_us": float(d["gpu__time_duration.sum"][0].replace(",", ""))} for d in res]
    js = {"round": rnd, "captures": summary}
    fwd = [d for d in summary.get("prof_fwd", []) if "band_u" in d["kernel"]] or summary.get("prof_fwd", [])
    if fwd:
        js["dominant_kernel_dram_bytes_per_launch"] = fwd[0]["dram_bytes"]
        js["dominant_kernel"] = fwd[0]["kernel"]
    json.dump(js, open(os.path.join(pdir, "ncu_summary.json"), "w"), indent=1)
    print("\n".join(lines))
    print(json.dumps(js, indent=1)[:2000])


if __name__ == "__main__":
    main()
