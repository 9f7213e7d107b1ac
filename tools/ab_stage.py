"""A/B of the collapsed path's stages between two builds of liblfm on one box: median device time of
lfm_A_stage FWD_T / ADJ_T (band_u) and of a full A_forward / A_adjoint of camera 0 and 1 of the 128^3 two-camera
config, L2 flushed before each launch.  Only the C ABI common to both builds is called.

    python tools/ab_stage.py LIB [LIB ...]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_03358_b200 import lfm  # noqa: E402  (structs and config marshalling only)
from workloads import flame_volume, make_config, uniform_vector  # noqa: E402


def run(path):
    lib = ctypes.CDLL(path)
    P, I, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    lib.lfm_plan_create.argtypes = [ctypes.POINTER(lfm.Geometry), I, ctypes.POINTER(P)]
    lib.lfm_plan_info.argtypes = [P, I, ctypes.POINTER(lfm.Info)]
    lib.lfm_A_stage.argtypes = [P, I, I, P, P, P, S, P]
    lib.lfm_A_forward.argtypes = [P, I, I, P, P, P, S, P]
    lib.lfm_A_adjoint.argtypes = [P, I, I, P, P, I, P, S, P]
    cfg = make_config("128^3 two-camera")
    vol = cfg["volume"]
    arr = (lfm.Camera * 2)(*[lfm._camera_struct(c) for c in cfg["cameras"]])
    g = lfm.Geometry(lfm.Volume(vol["nx"], vol["ny"], vol["nz"], vol["dx"], vol["dy"], vol["dz"]), 2, arr, 0)
    h = P()
    assert lib.lfm_plan_create(ctypes.byref(g), 0, ctypes.byref(h)) == 0
    inf = lfm.Info()
    lib.lfm_plan_info(h, 0, ctypes.byref(inf))
    ws = torch.empty(inf.ws_bytes, dtype=torch.uint8, device="cuda:0")
    x = torch.as_tensor(flame_volume(vol), device="cuda:0").reshape(-1)
    y = torch.empty(inf.n_pix, device="cuda:0")
    r = torch.as_tensor(uniform_vector(inf.n_pix, 1), device="cuda:0")
    gv = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, device="cuda:0")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: ctypes.c_void_p(t.data_ptr())

    def timed(fn, reps=21):
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
        return round(1e3 * sorted(out)[len(out) // 2], 2)

    res = {}
    for c in (0, 1):
        res["fwd_cam%d_us" % c] = timed(lambda: lib.lfm_A_forward(h, c, 1, p(x), p(y), p(ws), ws.numel(), st))
        res["adj_cam%d_us" % c] = timed(lambda: lib.lfm_A_adjoint(h, c, 1, p(r), p(gv), 0, p(ws), ws.numel(), st))
    lib.lfm_A_forward(h, 0, 1, p(x), p(y), p(ws), ws.numel(), st)
    res["band_u_fwd_us"] = timed(lambda: lib.lfm_A_stage(h, 0, 0, None, p(y), p(ws), ws.numel(), st))
    res["band_u_adj_us"] = timed(lambda: lib.lfm_A_stage(h, 0, 1, p(r), None, p(ws), ws.numel(), st))
    return res


if __name__ == "__main__":
    for path in sys.argv[1:]:
        print(json.dumps({"lib": path, **run(path)}), flush=True)
