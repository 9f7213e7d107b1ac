"""HBM read-only, write-only and copy bandwidth on this GPU (1 GiB buffers, CUDA events, best of 10): the
denominators behind the write-bound kernels (band_v forward writes U, band_u adjoint writes Z).  One JSON line."""
import json

import torch


def best(fn, reps=10):
    t = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t = min(t, a.elapsed_time(b))
    return t * 1e-3


n = 1 << 28  # 1 GiB of fp32
x = torch.rand(n, device="cuda")
y = torch.empty_like(x)
out = torch.empty((), device="cuda")
r = best(lambda: torch.sum(x, dim=0, out=out))
w = best(lambda: y.fill_(1.0))
c = best(lambda: y.copy_(x))
print(json.dumps({"bytes": 4 * n, "read_gbs": 4 * n / r / 1e9, "write_gbs": 4 * n / w / 1e9,
                  "copy_gbs_read_plus_write": 8 * n / c / 1e9}))
