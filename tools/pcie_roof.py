"""The host <-> device copy roof of bench.py's e2e line: pinned-memory H2D alone, D2H alone, and both directions at
once on two streams, for the pair's 40 MiB in + 40 MiB out (x 8 MiB + r_c 2 x 16 MiB; y_c 2 x 16 MiB + g 8 MiB at
128^3 two-camera), CUDA events, best of 20.  Prints one JSON line.

    python tools/pcie_roof.py
"""
import json

import torch


def main():
    n = (8 + 32) << 20  # bytes each way per pair
    h_in = torch.empty(n // 4).pin_memory()
    h_out = torch.empty(n // 4).pin_memory()
    d_in = torch.empty(n // 4, device="cuda")
    d_out = torch.empty(n // 4, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=20):
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_stream(torch.cuda.current_stream())
            s2.wait_stream(torch.cuda.current_stream())
            fn()
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"bytes_each_way": n, "h2d_ms": t_in, "d2h_ms": t_out, "both_ms": t_both,
                      "h2d_gbs": n / t_in / 1e6, "d2h_gbs": n / t_out / 1e6, "both_gbs_each_way": n / t_both / 1e6,
                      "pair_e2e_roof_pairs_per_s": 1e3 / t_both}))


if __name__ == "__main__":
    main()
