"""Thin ctypes binding of liblfm (include/lfm.h): argument marshalling only.

Every function has the C name without the `lfm_` prefix and takes torch CUDA tensors (fp32) for
device buffers; the stream defaults to torch's current stream.  No compute happens here: every
step of the hot path runs in liblfm's kernels.  Importing this module raises if liblfm.so is
missing -- there is no CPU fallback.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LFM_LIB") or os.path.join(_HERE, "liblfm.so")  # LFM_LIB: experiment variants

PILLBOX, DIRAC = 0, 1
SINGLE, PLENOPTIC = 0, 1
FWD, ADJ = 0, 1
PER_VIEW, COLLAPSED = 0, 1
MAJ_SUM, MAJ_FINISH = 1, 2
GRAD_ACCUMULATE = 2  # lfm_pwls_grad include_reg bit 1 (include/lfm.h)
STATUS = {0: "LFM_OK", 1: "LFM_E_INVALID", 2: "LFM_E_SINGULAR", 3: "LFM_E_DEGENERATE", 4: "LFM_E_MISMATCH",
          5: "LFM_E_ZERO_DATA", 6: "LFM_E_NONFINITE", 7: "LFM_E_CUDA", 8: "LFM_E_NOMEM"}
TAB = dict(S1F_START=0, S1F_LEN=1, S1F_W64=2, S1A_START=3, S1A_LEN=4, S1A_W64=5, S3F_START=6, S3F_LEN=7,
           S3F_W64=8, S3A_START=9, S3A_LEN=10, S3A_W64=11, CF_START=12, CF_LEN=13, CF_W64=14, ROT_MLO=15,
           ROT_W64=16, SCALARS=17)


class LfmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class Volume(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dz", ctypes.c_double)]


class Camera(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("basis", ctypes.c_int), ("f_main", ctypes.c_double),
                ("ap_s", ctypes.c_double), ("ap_t", ctypes.c_double), ("d_scene", ctypes.c_double),
                ("k_s", ctypes.c_int), ("k_t", ctypes.c_int), ("d_det", ctypes.c_double),
                ("d_mu_m", ctypes.c_double), ("d_d_mu", ctypes.c_double), ("f_mu", ctypes.c_double),
                ("fill", ctypes.c_double), ("nl_s", ctypes.c_int), ("nl_t", ctypes.c_int), ("n_a", ctypes.c_int),
                ("n_s", ctypes.c_int), ("n_t", ctypes.c_int), ("px_s", ctypes.c_double), ("px_t", ctypes.c_double),
                ("R", ctypes.c_double * 9), ("lens_layout", ctypes.c_int), ("aperture", ctypes.c_int)]


class Geometry(ctypes.Structure):
    _fields_ = [("vol", Volume), ("n_cam", ctypes.c_int), ("cam", ctypes.POINTER(Camera)), ("n_subsets", ctypes.c_int)]


class Info(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("basis", ctypes.c_int), ("nx", ctypes.c_int), ("ny", ctypes.c_int),
                ("nz", ctypes.c_int), ("n_vox", ctypes.c_longlong), ("n_s", ctypes.c_int), ("n_t", ctypes.c_int),
                ("n_pix", ctypes.c_longlong), ("k_s", ctypes.c_int), ("k_t", ctypes.c_int),
                ("n_views", ctypes.c_int), ("n_as", ctypes.c_int), ("n_at", ctypes.c_int),
                ("plane_array", ctypes.c_int), ("plane_detector", ctypes.c_int),
                ("vox_r", ctypes.c_double * 3), ("rot_D", ctypes.c_double * 3), ("shear", ctypes.c_double * 6),
                ("rot_passes", ctypes.c_int), ("rot_perm", ctypes.c_int * 9), ("taps_s1", ctypes.c_int), ("taps_s3", ctypes.c_int),
                ("taps_c", ctypes.c_int), ("ws_bytes", ctypes.c_size_t), ("table_bytes", ctypes.c_size_t),
                ("fma_alg", ctypes.c_double * 2), ("bytes_alg", ctypes.c_double * 2),
                ("fma_stage", ctypes.c_double * 2), ("mma_stage", ctypes.c_double * 2),
                ("kind_stage", ctypes.c_int * 2), ("fma_spass", ctypes.c_double * 2),
                ("subset_collapsed", ctypes.c_int), ("s3_terms", ctypes.c_int),
                ("f16_stage", ctypes.c_int * 2)]

    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if hasattr(v, "__len__") else v
        return out


if not os.path.exists(LIB_PATH):
    raise ImportError("liblfm.so not built (%s): run `python -m paper_1812_03358_b200.build` "
                      "(there is no CPU fallback)" % LIB_PATH)
_lib = ctypes.CDLL(LIB_PATH)
_P = ctypes.c_void_p
_I = ctypes.c_int
_S = ctypes.c_size_t
_D = ctypes.c_double
_F = ctypes.c_float
_PP = ctypes.POINTER(ctypes.c_void_p)
_SIGS = {
    "lfm_plan_create": [ctypes.POINTER(Geometry), _I, ctypes.POINTER(_P)],
    "lfm_plan_destroy": [_P],
    "lfm_plan_info": [_P, _I, ctypes.POINTER(Info)],
    "lfm_plan_export_table": [_P, _I, _I, _I, _I, _P, _S, ctypes.POINTER(_S)],
    "lfm_lf_transport": [_P, _I, _I, _I, _P, _P, _P, _S, _P],
    "lfm_vol_rotate": [_P, _I, _I, _P, _P, _I, _P, _S, _P],
    "lfm_vol_accumulate": [_P, _P, ctypes.c_longlong, _P],
    "lfm_A_forward": [_P, _I, _I, _P, _P, _P, _S, _P],
    "lfm_A_adjoint": [_P, _I, _I, _P, _P, _I, _P, _S, _P],
    "lfm_A_forward_rows": [_P, _I, _I, _I, _I, _P, _P, _P, _S, _P],
    "lfm_A_adjoint_rows": [_P, _I, _I, _I, _I, _P, _P, _I, _P, _S, _P],
    "lfm_A_forward_window": [_P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _S, _P],
    "lfm_A_adjoint_window": [_P, _I, _I, _I, _I, _I, _I, _P, _P, _I, _P, _S, _P],
    "lfm_A_stage": [_P, _I, _I, _P, _P, _P, _S, _P],
    "lfm_A_forward_subset": [_P, _I, _I, _P, _P, _P, _S, _P],
    "lfm_A_adjoint_subset": [_P, _I, _I, _P, _P, _I, _P, _S, _P],
    "lfm_pwls_stats": [_P, _I, _P, _P, _P, _P, _P, _S, _P],
    "lfm_pwls_gains": [_P, _P, _P, _P, _P],
    "lfm_pwls_grad": [_P, _I, _I, _I, _I, _P, _PP, _PP, _PP, _P, _F, _F, _I, _P, _P, _P, _S, _P],
    "lfm_majoriser": [_P, _I, _I, _I, _PP, _F, _I, _P, _P, _S, _P],
    "lfm_fista_update": [_P, _P, _P, _P, _P, _D, _D, _P],
    "lfm_last_launch_count": [],
    "lfm_last_error": [],
    "lfm_version": [],
}
for _name, _args in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _I
_lib.lfm_last_error.restype = ctypes.c_char_p
_lib.lfm_version.restype = ctypes.c_char_p

EXPORTED = sorted(_SIGS)


def _check(status):
    if status != 0:
        raise LfmError(status, _lib.lfm_last_error().decode())


def version():
    return _lib.lfm_version().decode()


def last_launch_count():
    return _lib.lfm_last_launch_count()


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(int(t))


def _stream(stream):
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _camera_struct(c):
    cs = Camera()
    for name, _ in Camera._fields_:
        if name == "R":
            cs.R = (ctypes.c_double * 9)(*[float(v) for v in c["R"]])
        elif name in ("lens_layout", "aperture"):
            setattr(cs, name, int(c.get(name, 0)))
        else:
            setattr(cs, name, c[name])
    return cs


class Plan:
    """Owns an lfm_plan built from a workloads-style config dict {volume, cameras}."""

    def __init__(self, config, device=0, n_subsets=0):
        vol = config["volume"]
        cams = config["cameras"]
        arr = (Camera * len(cams))(*[_camera_struct(c) for c in cams])
        g = Geometry(Volume(vol["nx"], vol["ny"], vol["nz"], vol["dx"], vol["dy"], vol["dz"]), len(cams), arr,
                     int(n_subsets))
        self.n_subsets = int(n_subsets) if n_subsets > 1 else 0
        h = _P()
        _check(_lib.lfm_plan_create(ctypes.byref(g), int(device), ctypes.byref(h)))
        self._h = h
        self.device = device
        self.n_cam = len(cams)
        self.config = config
        self.infos = [self.info(c) for c in range(self.n_cam)]
        self.ws_bytes = self.infos[0]["ws_bytes"]

    @property
    def handle(self):
        return self._h

    def info(self, cam):
        inf = Info()
        _check(_lib.lfm_plan_info(self._h, cam, ctypes.byref(inf)))
        return inf.as_dict()

    def export_table(self, cam, table, axis=0, index=0):
        import numpy as np
        tid = TAB[table] if isinstance(table, str) else table
        need = ctypes.c_size_t(0)
        _check(_lib.lfm_plan_export_table(self._h, cam, tid, axis, index, None, 0, ctypes.byref(need)))
        name = table if isinstance(table, str) else ""
        dtype = np.int32 if (name.endswith("START") or name.endswith("LEN") or name.endswith("MLO")) else np.float64
        out = np.zeros(need.value // np.dtype(dtype).itemsize, dtype)
        _check(_lib.lfm_plan_export_table(self._h, cam, tid, axis, index,
                                          out.ctypes.data_as(ctypes.c_void_p), need.value, None))
        return out

    def workspace(self):
        return torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda:%d" % self.device)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lfm_plan_destroy(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- the C-ABI calls, same names ------------------------------------------------------------
def lf_transport(plan, cam, dst_plane, src_plane, src, dst, ws, stream=None):
    _check(_lib.lfm_lf_transport(plan.handle, cam, dst_plane, src_plane, _ptr(src), _ptr(dst), _ptr(ws),
                                 ws.numel(), _stream(stream)))


def vol_rotate(plan, cam, direction, src, dst, ws, accumulate=False, stream=None):
    _check(_lib.lfm_vol_rotate(plan.handle, cam, direction, _ptr(src), _ptr(dst), int(accumulate), _ptr(ws),
                               ws.numel(), _stream(stream)))


def vol_accumulate(src, dst, stream=None):
    """dst += src (the camera sum of concurrent backprojections)."""
    _check(_lib.lfm_vol_accumulate(_ptr(src), _ptr(dst), int(src.numel()), _stream(stream)))


def A_forward(plan, cam, x, y, ws, path=COLLAPSED, stream=None):
    _check(_lib.lfm_A_forward(plan.handle, cam, path, _ptr(x), _ptr(y), _ptr(ws), ws.numel(), _stream(stream)))


def A_adjoint(plan, cam, y, x, ws, accumulate=False, path=COLLAPSED, stream=None):
    _check(_lib.lfm_A_adjoint(plan.handle, cam, path, _ptr(y), _ptr(x), int(accumulate), _ptr(ws), ws.numel(),
                              _stream(stream)))


def A_forward_rows(plan, cam, row0, row1, x, y, ws, path=COLLAPSED, stream=None):
    _check(_lib.lfm_A_forward_rows(plan.handle, cam, path, row0, row1, _ptr(x), _ptr(y), _ptr(ws), ws.numel(),
                                   _stream(stream)))


def A_forward_window(plan, cam, row0, row1, col0, col1, x, y, ws, path=COLLAPSED, stream=None):
    _check(_lib.lfm_A_forward_window(plan.handle, cam, path, row0, row1, col0, col1, _ptr(x), _ptr(y), _ptr(ws),
                                     ws.numel(), _stream(stream)))


def A_adjoint_window(plan, cam, row0, row1, col0, col1, y, x, ws, accumulate=False, path=COLLAPSED, stream=None):
    _check(_lib.lfm_A_adjoint_window(plan.handle, cam, path, row0, row1, col0, col1, _ptr(y), _ptr(x), int(accumulate),
                                     _ptr(ws), ws.numel(), _stream(stream)))


def A_forward_subset(plan, cam, subset, x, y, ws, stream=None):
    """y = (K/|S_m|) sum_{k in S_m} A_ck x over the plan's view subset m (include/lfm.h)."""
    _check(_lib.lfm_A_forward_subset(plan.handle, cam, subset, _ptr(x), _ptr(y), _ptr(ws), ws.numel(), _stream(stream)))


def A_adjoint_subset(plan, cam, subset, y, x, ws, accumulate=False, stream=None):
    _check(_lib.lfm_A_adjoint_subset(plan.handle, cam, subset, _ptr(y), _ptr(x), int(accumulate), _ptr(ws), ws.numel(),
                                     _stream(stream)))


STAGE_FWD_T, STAGE_ADJ_T, STAGE_FWD_S, STAGE_ADJ_S = 0, 1, 2, 3


def A_stage(plan, cam, stage, inp, out, ws, stream=None):
    """One kernel of the collapsed two-pass path on the workspace intermediate (include/lfm.h)."""
    _check(_lib.lfm_A_stage(plan.handle, cam, stage, _ptr(inp), _ptr(out), _ptr(ws), ws.numel(), _stream(stream)))


def A_adjoint_rows(plan, cam, row0, row1, y, x, ws, accumulate=False, path=COLLAPSED, stream=None):
    _check(_lib.lfm_A_adjoint_rows(plan.handle, cam, path, row0, row1, _ptr(y), _ptr(x), int(accumulate), _ptr(ws),
                                   ws.numel(), _stream(stream)))


def pwls_stats(plan, cam, Ax, y, w, stats3, ws, stream=None):
    _check(_lib.lfm_pwls_stats(plan.handle, cam, _ptr(Ax), _ptr(y), _ptr(w), _ptr(stats3), _ptr(ws), ws.numel(),
                               _stream(stream)))


def pwls_gains(plan, stats, gamma, flag=None, stream=None):
    _check(_lib.lfm_pwls_gains(plan.handle, _ptr(stats), _ptr(gamma), _ptr(flag), _stream(stream)))


def _ptr_array(ts, n):
    arr = (ctypes.c_void_p * n)()
    for i, t in enumerate(ts):
        arr[i] = None if t is None else t.data_ptr()
    return arr


def pwls_grad(plan, x, ys, ws_, Axs, gamma, beta, nu, grad, ws, cam0=0, cam1=None, include_reg=True, cost=None,
              path=COLLAPSED, stream=None, subset=-1):
    n = plan.n_cam
    cam1 = n if cam1 is None else cam1
    _check(_lib.lfm_pwls_grad(plan.handle, path, int(subset), cam0, cam1, _ptr(x), _ptr_array(ys, n), _ptr_array(ws_, n),
                              _ptr_array(Axs, n), _ptr(gamma), float(beta), float(nu), int(include_reg), _ptr(grad),
                              _ptr(cost), _ptr(ws), ws.numel(), _stream(stream)))


def majoriser(plan, weights, beta, d, ws, cam0=0, cam1=None, mode=MAJ_SUM | MAJ_FINISH, path=COLLAPSED,
              stream=None):
    n = plan.n_cam
    cam1 = n if cam1 is None else cam1
    _check(_lib.lfm_majoriser(plan.handle, path, cam0, cam1, _ptr_array(weights, n), float(beta), int(mode), _ptr(d),
                              _ptr(ws), ws.numel(), _stream(stream)))


def fista_update(plan, x, z, grad, d, t_old, t_new, stream=None):
    _check(_lib.lfm_fista_update(plan.handle, _ptr(x), _ptr(z), _ptr(grad), _ptr(d), float(t_old), float(t_new),
                                 _stream(stream)))
