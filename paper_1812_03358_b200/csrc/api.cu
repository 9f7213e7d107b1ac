// liblfm C ABI (include/lfm.h): argument validation, workspace layout, and the composition of
// kernels into the paper's operators.  Every step of the hot path runs in kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "lfm_internal.h"
#include "lfm_kernels.h"

namespace lfm {
lfm_status cuda_check(cudaError_t e, const char* what, std::string& err);
}

using namespace lfm;

namespace {
thread_local std::string g_err;
thread_local int g_last_launches = 0;

lfm_status fail(lfm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

// Apply calls run on the plan's device: switch to it for the call (kernel attributes, SM counts and tensor maps
// are per device) and restore the caller's current device afterwards.
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const lfm_plan_s* p) {
    if (!p || p->device < 0) return;
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) { cudaGetLastError(); return; }
    if (cur != p->device && cudaSetDevice(p->device) == cudaSuccess) prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct WsLayout {
  size_t r0, r1, xt, f, s, s2, z, zt, p, am, h16, rs, cs, total;
};

WsLayout layout(const lfm_plan_s* p) {
  size_t V = 0, F = 0, S = 0, Z = 0, P = 0, R = 0, C = 0;
  for (const CameraPlan& c : p->cams) {
    C = std::max(C, (size_t)((c.info.n_s + 255) / 256 * 256) * 4);
    P = std::max(P, (size_t)c.info.n_pix * 4);
    R = std::max(R, (size_t)c.info.ny * c.info.nz * 4);
    V = std::max(V, (size_t)c.info.n_vox * 4);
    F = std::max(F, c.ws_fields);
    Z = std::max(Z, c.ws_z);
    S = std::max(S, (size_t)std::max<long long>(c.info.n_pix, c.info.n_vox) * 4);
  }
  WsLayout L;
  L.r0 = 0;
  L.r1 = L.r0 + al256(V);
  L.xt = L.r1 + al256(V);
  L.f = L.xt + al256(V);
  L.s = L.f + al256(F);
  L.s2 = L.s + al256(S);
  L.z = L.s2 + al256(S);
  L.zt = L.z + al256(Z);
  L.p = L.zt + al256(Z);
  L.am = L.p + al256(4096 * 8 * 4);
  L.h16 = L.am + al256(LFM_AMAX_SLOTS * 4);
  L.rs = L.h16 + al256(P);
  L.cs = L.rs + al256(R);
  L.total = L.cs + al256(C);
  return L;
}

struct Ws {
  float *r0, *r1, *xt, *f, *s, *s2, *z, *zt;
  double* p;
  float* am;      // partial maxima of the 2xFP16 t-pass input's source: of x^r (forward), of y (adjoint)
  uint16_t* h16;  // fp16 hi (n_pix) then lo (n_pix) of 2^e y: the adjoint t pass input in the 2xFP16 form
  float* rs;      // per-row inverse scales of the row-scaled fp16 split of x^r (nz ny)
  float* cs;      // per-column inverse scales of the column-scaled fp16 split of y (n_s rounded up to 256)
};

lfm_status get_ws(const lfm_plan_s* p, void* ws, size_t ws_bytes, Ws& w) {
  WsLayout L = layout(p);
  if (!ws) return fail(LFM_E_INVALID, "workspace pointer is NULL");
  if (ws_bytes < L.total) return fail(LFM_E_INVALID, "workspace too small: need " + std::to_string(L.total) + " bytes");
  if (((uintptr_t)ws & 255) != 0) return fail(LFM_E_INVALID, "workspace must be 256-byte aligned");
  char* b = (char*)ws;
  w.r0 = (float*)(b + L.r0);
  w.r1 = (float*)(b + L.r1);
  w.f = (float*)(b + L.f);
  w.s = (float*)(b + L.s);
  w.s2 = (float*)(b + L.s2);
  w.z = (float*)(b + L.z);
  w.xt = (float*)(b + L.xt);
  w.zt = (float*)(b + L.zt);
  w.p = (double*)(b + L.p);
  w.am = (float*)(b + L.am);
  w.h16 = (uint16_t*)(b + L.h16);
  w.rs = (float*)(b + L.rs);
  w.cs = (float*)(b + L.cs);
  return LFM_OK;
}

lfm_status check_cam(const lfm_plan_s* p, int cam, bool need_device = true) {
  if (!p) return fail(LFM_E_INVALID, "plan is NULL");
  if (cam < 0 || cam >= (int)p->cams.size()) return fail(LFM_E_INVALID, "camera index out of range");
  if (need_device && p->device < 0) return fail(LFM_E_INVALID, "host-only plan (created with cuda_device = -1)");
  return LFM_OK;
}

#define TRY(expr)                         \
  do {                                    \
    std::string _e;                       \
    lfm_status _s = (expr);               \
    (void)_e;                             \
    if (_s != LFM_OK) return _s;          \
  } while (0)

// Rotation forward: returns the buffer holding x^r (x itself if the pose is the identity).  Stages in
// order: the quarter-turn relabelling (if any, reading R7), then the active shear passes z, x, y;
// intermediate results ping-pong between w.r0 and w.r1, the last one goes to final_out if given.
lfm_status rotate_fwd(const CameraPlan& cp, const float* x, float* final_out, int accumulate, const Ws& w,
                      void* stream, const float** xr) {
  int act[4], na = 0;
  if (cp.has_perm) act[na++] = -1;
  for (int q = 0; q < 3; ++q)
    if (cp.rot[q].active) act[na++] = q;
  const float* cur = x;
  std::string err;
  for (int i = 0; i < na; ++i) {
    bool last = i == na - 1;
    float* dst = (last && final_out) ? final_out : ((cur == w.r0) ? w.r1 : w.r0);
    const int acc = (last && final_out) ? accumulate : 0;
    lfm_status st = act[i] < 0 ? k_permute(cur, dst, cp.info.nx, cp.info.ny, cp.info.nz, cp.perm_axis[0],
                                           cp.perm_sign[0], acc, stream, err)
                               : launch_shear(cp.rot[act[i]], 0, cur, dst, cp.info.nx, cp.info.ny, cp.info.nz, acc,
                                              stream, err);
    if (st != LFM_OK) return fail(st, err);
    cur = dst;
  }
  if (na == 0 && final_out) {
    lfm_status st = k_copy_scale(x, final_out, cp.info.n_vox, 1.f, accumulate, stream, err);
    if (st != LFM_OK) return fail(st, err);
    cur = final_out;
  }
  *xr = cur;
  return LFM_OK;
}

// Rotation adjoint E^zT E^xT E^yT, then the inverse relabelling P^T, applied to `in`, written (or
// accumulated) into `out`.  `in` may be w.r0 or w.r1 (the ping-pong never writes the buffer it reads).
lfm_status rotate_adj(const CameraPlan& cp, const float* in, float* out, int accumulate, const Ws& w, void* stream) {
  int act[4], na = 0;
  for (int q = 2; q >= 0; --q)
    if (cp.rot[q].active) act[na++] = q;
  if (cp.has_perm) act[na++] = -1;
  std::string err;
  if (na == 0) {
    lfm_status st = k_copy_scale(in, out, cp.info.n_vox, 1.f, accumulate, stream, err);
    return st == LFM_OK ? st : fail(st, err);
  }
  const float* cur = in;
  for (int i = 0; i < na; ++i) {
    bool last = i == na - 1;
    float* dst = last ? out : ((cur == w.r0) ? w.r1 : w.r0);
    const int acc = last ? accumulate : 0;
    lfm_status st = act[i] < 0 ? k_permute(cur, dst, cp.info.nx, cp.info.ny, cp.info.nz, cp.perm_axis[1],
                                           cp.perm_sign[1], acc, stream, err)
                               : launch_shear(cp.rot[act[i]], 1, cur, dst, cp.info.nx, cp.info.ny, cp.info.nz, acc,
                                              stream, err);
    if (st != LFM_OK) return fail(st, err);
    cur = dst;
  }
  return LFM_OK;
}

lfm_status sep(const SepOp& op, const float* src, float* out, int b0, int n_out, int acc, void* stream,
               int out_r0 = 0, int out_r1 = -1, int win_r0 = 0, int win_r1 = -1, int out_c0 = 0, int out_c1 = -1,
               float* part = nullptr, size_t part_bytes = 0, F16Src amx = F16Src()) {
  std::string err;
  lfm_status st = launch_sep(op, src, out, b0, n_out, acc, stream, err, out_r0, out_r1, win_r0, win_r1, out_c0, out_c1,
                             part, part_bytes, amx);
  return st == LFM_OK ? st : fail(st, err);
}

// A detector window [r0, r1) x [c0, c1) (multi-GPU shards; r1 / c1 < 0 = to the end).
struct Win {
  int r0 = 0, r1 = -1, c0 = 0, c1 = -1;
  bool cols(int n_s) const { return c0 > 0 || (c1 >= 0 && c1 < n_s); }
};

// 2xFP16 form of the tcgen05 t passes (band_u_kernel<., true>): the t-pass input is written pre-split into fp16
// hi + lo by its producer (band_v forward / split16_kernel), scaled by 2^e from the maxima of its source (DESIGN
// §6).  Default wherever the plan has the fp16 images and the detector rows are 16-byte aligned in fp16;
// LFM_UMMA_TF32=1 selects the 3xTF32 form (A/B, tests).
static bool f16_env() {
  static const bool off = std::getenv("LFM_UMMA_TF32") != nullptr;
  return !off;
}
static bool f16_fwd(const CameraPlan& cp, const SepOp& c2) {
  return f16_env() && cp.fwd_split && cp.fwd_t == 3 && c2.kind == 8 && c2.ft->d_uh && cp.info.n_s % 8 == 0;
}
static bool f16_adj(const CameraPlan& cp, const SepOp& c1) {
  return f16_env() && c1.kind == 8 && c1.ft->d_uh && cp.info.n_s % 8 == 0;
}

// One term of the collapsed forward: band_v s pass (T) into U, band_u t pass (c2) into y.  2xFP16: the maxima of
// x^r (computed once per call, `amax_done`) set the scale with which band_v writes U as fp16 hi / lo.
static lfm_status vt_forward(const CameraPlan& cp, const VTab& T, const SepOp& c2, const float* xr, float* y, int acc,
                             const Ws& w, void* stream, Win win, bool& amax_done) {
  std::string err;
  lfm_status st;
  if (f16_fwd(cp, c2)) {
    // x^r pre-split into fp16 hi / lo (w.xt) when band_v has its fp16 images: no split warps in either kernel
    static const bool no_x16 = std::getenv("LFM_NO_X16") != nullptr;  // A/B: band_v splits x^r itself
    uint16_t* x16 = T.d_h16 && T.BK == 32 && !no_x16 ? reinterpret_cast<uint16_t*>(w.xt) : nullptr;
    if (x16 && cp.info.nx % 8) x16 = nullptr;  // fp16 rows of x^r must start on 16-byte boundaries
    if (!amax_done) {  // one pass: row-scaled split (x16) and the maxima of x^r, or the maxima alone
      st = x16 ? k_split16_rows(xr, cp.info.ny * cp.info.nz, cp.info.nx, w.am, w.rs, x16, x16 + cp.info.n_vox, stream, err)
               : k_amax(xr, cp.info.n_vox, w.am, stream, err);
      if (st != LFM_OK) return fail(st, err);
    }
    amax_done = true;
    if ((st = k_vpass_fwd(cp, T, xr, w.z, stream, err, win.c0, win.c1, w.am, x16, w.rs)) != LFM_OK) return fail(st, err);
    F16Src h;
    h.hi = reinterpret_cast<const uint16_t*>(w.z);
    h.lo = h.hi + (size_t)cp.cf[0].n_rows * cp.info.nz * cp.info.ny;
    h.amax = w.am;
    h.amax_scale = T.lsum;
    return sep(c2, w.z, y, 0, 1, acc, stream, win.r0, win.r1, 0, -1, win.c0, win.c1, w.zt, cp.ws_z, h);
  }
  if ((st = k_vpass_fwd(cp, T, xr, w.z, stream, err, win.c0, win.c1)) != LFM_OK) return fail(st, err);
  return sep(c2, w.z, y, 0, 1, acc, stream, win.r0, win.r1, 0, -1, win.c0, win.c1, w.zt, cp.ws_z);
}

// the adjoint t pass's input split with a scale per detector column in one kernel (k_split16_cols) instead of
// the global maxima + split (two kernels); LFM_SPLIT_GLOBAL=1 keeps the latter (A/B)
static bool cols_split() {
  static const bool off = std::getenv("LFM_SPLIT_GLOBAL") != nullptr;
  return !off;
}

// The PWLS residual r = w (Ax - gamma[cam] y) as the adjoint's input, computed inside the t pass's input split
// (lfm_pwls_grad passes it instead of a materialised r when that split is the column-scaled one, see res_fusable)
struct ResSrc {
  const float* Ax;
  const float* y;
  const float* w;
  const double* gamma;
  int cam;
};
static bool al16p(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

// The adjoint t pass (c1) of y's rows [r0, r1): 2xFP16 = fp16 hi / lo of y (scaled per column, or by 2^e from the
// maxima of those rows) into w.h16 -- done once per call and kind (`split_state`: 0 none, 1 global scale, 2 column
// scales), then band_u from them.  res != nullptr: y is the residual of *res (only with column scales).
static lfm_status t_adjoint(const CameraPlan& cp, const SepOp& c1, const float* y, const Ws& w, void* stream, Win win,
                            int& split_state, bool z16 = false, const ResSrc* res = nullptr) {
  if (!f16_adj(cp, c1)) {
    if (res) return fail(LFM_E_INVALID, "internal: fused residual without the 2xFP16 t pass");
    return sep(c1, y, w.z, 0, 1, 0, stream, 0, -1, win.r0, win.r1, win.c0, win.c1);
  }
  const int n_s = cp.info.n_s, r0 = std::max(0, win.r0), r1 = win.r1 < 0 ? cp.info.n_t : std::min(win.r1, cp.info.n_t);
  const size_t np = (size_t)cp.info.n_pix;
  // column scales: with the fp16 Z output only (band_u's OUT16 epilogue applies them), 16-byte aligned rows of y
  // (n_s % 8 == 0 already holds for the 2xFP16 form)
  const bool cs = cols_split() && z16 && (res ? al16p(res->Ax) && al16p(res->y) && al16p(res->w) : al16p(y));
  if (res && !cs) return fail(LFM_E_INVALID, "internal: fused residual without the column-scaled split");
  const int need = cs ? 2 : 1;
  if (split_state != need && r1 > r0) {
    std::string err;
    const long long off = (long long)r0 * n_s, n = (long long)(r1 - r0) * n_s;
    lfm_status st;
    if (cs && res) {
      st = k_split16_cols_residual(res->Ax + off, res->y + off, res->w + off, res->gamma, res->cam, r1 - r0, n_s,
                                   (n_s + 255) / 256 * 256, w.am, w.cs, w.h16 + off, w.h16 + np + off, stream, err);
    } else if (cs) {
      st = k_split16_cols(y + off, r1 - r0, n_s, (n_s + 255) / 256 * 256, w.am, w.cs, w.h16 + off, w.h16 + np + off,
                          stream, err);
    } else {
      st = k_amax(y + off, n, w.am, stream, err);
      if (st == LFM_OK) st = k_split16(y + off, n, w.am, w.h16 + off, w.h16 + np + off, stream, err);
    }
    if (st != LFM_OK) return fail(st, err);
  }
  split_state = need;
  F16Src h;
  h.hi = w.h16;
  h.lo = w.h16 + np;
  h.amax = w.am;
  if (cs) h.cinv = w.cs;
  if (z16) {  // Z as fp16 hi / lo of 2^e' Z for band_v's 2xFP16 form (k_vpass_adj with in_scale = u_lsum)
    h.out_hi = reinterpret_cast<uint16_t*>(w.z);
    h.out_lo = h.out_hi + (size_t)c1.n_ot * c1.n_os;
    h.out_scale16 = c1.ft->u_lsum;
  }
  return sep(c1, y, w.z, 0, 1, 0, stream, 0, -1, win.r0, win.r1, win.c0, win.c1, nullptr, 0, h);
}

// the adjoint's t pass can hand band_v an fp16 Z (every term's tables have the 2xFP16 forms)
static bool z16_ok(const CameraPlan& cp, const SepOp& c1, const VTab& va);
static int eff_path(const CameraPlan& cp, int path);
// lfm_pwls_grad may fuse the residual into the adjoint's input split: the camera's whole adjoint runs the
// collapsed tcgen05 path with the column-scaled split in every term (LFM_NO_FUSED_RES=1: the residual kernel first)
static bool res_fusable(const CameraPlan& cp, int path, const float* Ax, const float* y, const float* wv) {
  if (std::getenv("LFM_NO_FUSED_RES") || eff_path(cp, path) != LFM_PATH_COLLAPSED || !cols_split()) return false;
  if (!(al16p(Ax) && al16p(y) && al16p(wv))) return false;
  if (!f16_adj(cp, cp.adj_c1) || !z16_ok(cp, cp.adj_c1, cp.va)) return false;
  for (const Component& cm : cp.comps)
    if (!f16_adj(cp, cm.adj_c1) || !z16_ok(cp, cm.adj_c1, cm.va)) return false;
  return true;
}

// the adjoint's t pass can hand band_v an fp16 Z (every term's tables have the 2xFP16 forms)
static bool z16_ok(const CameraPlan& cp, const SepOp& c1, const VTab& va) {
  static const bool no_z16 = std::getenv("LFM_NO_Z16") != nullptr;  // A/B: fp32 Z, band_v splits it
  return f16_adj(cp, c1) && cp.adj_t == 3 && vpass_adj_in16(va) && !no_z16;
}

// the collapsed path runs on the tcgen05 kernels end to end (band_v s passes, band_u t passes), the form whose
// kernels restrict themselves to a column window
static bool tc_two_pass(const CameraPlan& cp) {
  bool ok = cp.fwd_split && cp.fwd_t == 3 && cp.adj_t == 3 && cp.fwd_c2.kind == 8 && cp.adj_c1.kind == 8;
  for (const Component& cm : cp.comps) ok = ok && cm.fwd_c2.kind == 8 && cm.adj_c1.kind == 8 && cm.vf.d_img && cm.va.d_img;
  return ok;
}

// The collapsed path of a non-separable lenslet stage (T > 1 terms) exists only as the tcgen05 two-pass form (a
// sum over terms of s pass + t pass); without it such a camera's collapsed requests run on the per-view path.
static int eff_path(const CameraPlan& cp, int path) {
  return (path == LFM_PATH_COLLAPSED && !cp.comps.empty() && !tc_two_pass(cp)) ? LFM_PATH_PER_VIEW : path;
}

// y on the window rows [r0, r1) x columns [c0, c1) of A_c x.  Other entries of partially covered tiles may be
// written (with their correct values); the column window only saves work on the tcgen05 path (band_v items of
// the window's 256-column tiles; band_u items of those tiles, split-K when few).
lfm_status forward_impl(const CameraPlan& cp, int path, const float* x, float* y, const Ws& w, void* stream,
                        Win win = Win()) {
  const int r0 = win.r0, r1 = win.r1;
  path = eff_path(cp, path);
  const float* xr;
  TRY(rotate_fwd(cp, x, nullptr, 0, w, stream, &xr));
  const bool plen = cp.info.type == LFM_PLENOPTIC;
  if (path == LFM_PATH_COLLAPSED && !cp.comps.empty()) {
    // non-separable lenslet stage: y = sum over terms of (band_v s pass, band_u t pass), terms >= 1 accumulated
    bool amax_done = false;
    TRY(vt_forward(cp, cp.vf, cp.fwd_c2, xr, y, 0, w, stream, win, amax_done));
    for (const Component& cm : cp.comps) TRY(vt_forward(cp, cm.vf, cm.fwd_c2, xr, y, 1, w, stream, win, amax_done));
    return LFM_OK;
  }
  if (path == LFM_PATH_COLLAPSED) {
    if (cp.fwd_split) {
      if (cp.fwd_t == 3) {  // band_v on the tensor cores: slices -> interleaved U, then band_u
        bool amax_done = false;
        return vt_forward(cp, cp.vf, cp.fwd_c2, xr, y, 0, w, stream, win, amax_done);
      } else if (cp.fwd_t == 2) {
        // direct s pass (spass_fwd_kernel): slices -> interleaved U
        std::string err;
        lfm_status st = k_spass_fwd(cp, xr, w.z, stream, err);
        if (st != LFM_OK) return fail(st, err);
      } else if (cp.fwd_t) {
        // s pass as a t pass over the transposed slices, written back in the interleaved U layout
        const int nx = cp.info.nx, ny = cp.info.ny, nz = cp.info.nz;
        const long long nslice = (long long)nx * ny;
        std::string err;
        lfm_status st = k_transpose(xr, w.xt, nz, ny, nx, nslice, nx, nslice, ny, stream, err);
        if (st != LFM_OK) return fail(st, err);
        TRY(sep(cp.fwd_p1, w.xt, w.z, 0, nz, 0, stream));
      } else {
        TRY(sep(cp.fwd_c1, xr, w.z, 0, cp.info.nz, 0, stream));
      }
      return sep(cp.fwd_c2, w.z, y, 0, 1, 0, stream, r0, r1, 0, -1, win.c0, win.c1, w.zt, cp.ws_z);
    }
    return sep(cp.fwd_c, xr, y, 0, 1, 0, stream, r0, r1);
  }
  if (plen) {
    TRY(sep(cp.fwd_s1, xr, w.f, 0, cp.info.n_views, 0, stream));
    return sep(cp.fwd_s3, w.f, y, 0, 1, 0, stream, r0, r1);
  }
  return sep(cp.fwd_s1, xr, y, 0, 1, 0, stream, r0, r1);
}

// y (n_t x n_s) with zeros outside the window (the generic form of a column window)
__global__ void mask_window_kernel(const float* __restrict__ y, float* __restrict__ out, int n_t, int n_s, int r0, int r1,
                                   int c0, int c1) {
  const long long n = (long long)n_t * n_s;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / n_s), c = (int)(i % n_s);
    out[i] = (r >= r0 && r < r1 && c >= c0 && c < c1) ? y[i] : 0.f;
  }
}

// x (+)= A_c^T P y, P keeping the window rows [r0, r1) x columns [c0, c1) of y (others treated as zero).
lfm_status adjoint_impl(const CameraPlan& cp, int path, const float* y, float* x, int accumulate, const Ws& w,
                        void* stream, Win win = Win(), const ResSrc* res = nullptr) {
  int r0 = win.r0, r1 = win.r1;
  path = eff_path(cp, path);
  const bool rot = cp.info.rot_passes != 0;
  float* target = rot ? w.r0 : x;
  int acc = rot ? 0 : accumulate;
  const bool plen = cp.info.type == LFM_PLENOPTIC;
  const bool tc_cols = path == LFM_PATH_COLLAPSED && tc_two_pass(cp) && win.c0 % 4 == 0;
  if (win.cols(cp.info.n_s) && !tc_cols) {
    // kernels without column windows: mask y into scratch, then the row-windowed adjoint of the masked copy
    const int rr1 = r1 < 0 ? cp.info.n_t : r1, cc1 = win.c1 < 0 ? cp.info.n_s : win.c1;
    mask_window_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(y, w.s2, cp.info.n_t, cp.info.n_s, r0, rr1, win.c0, cc1);
    ++g_launches;
    y = w.s2;
    win.c0 = 0;
    win.c1 = -1;
  }
  if (path == LFM_PATH_COLLAPSED) {
    // one output: all (vt, n) rows; the column window selects the 256-column tiles of Z
    int split_state = 0;
    const bool z16 = z16_ok(cp, cp.adj_c1, cp.va) && win.c0 % 8 == 0;  // fp16 Z maps start on 16-byte boundaries
    TRY(t_adjoint(cp, cp.adj_c1, y, w, stream, win, split_state, z16, res));
    if (cp.adj_t == 2 || cp.adj_t == 3) {
      // direct s pass (spass_adj_kernel, or band_v on the tensor cores) on Z
      std::string err;
      lfm_status st = cp.adj_t == 3 ? k_vpass_adj(cp, cp.va, w.z, target, acc, stream, err, win.c0, win.c1,
                                                  z16 ? w.am : nullptr, cp.adj_c1.ft->u_lsum)
                                    : k_spass_adj(cp, w.z, target, acc, stream, err);
      if (st != LFM_OK) return fail(st, err);
      // non-separable lenslet stage: the other terms' t and s passes, accumulated (tcgen05 path only, eff_path)
      for (const Component& cm : cp.comps) {
        const bool zc = z16_ok(cp, cm.adj_c1, cm.va) && win.c0 % 8 == 0;
        TRY(t_adjoint(cp, cm.adj_c1, y, w, stream, win, split_state, zc, res));
        if ((st = k_vpass_adj(cp, cm.va, w.z, target, 1, stream, err, win.c0, win.c1, zc ? w.am : nullptr,
                              cm.adj_c1.ft->u_lsum)) != LFM_OK)
          return fail(st, err);
      }
    } else if (cp.adj_t) {
      // Z_n -> ZT_n = [j][vt] per slice, then the s pass as a t pass with transposed output into x_n
      const int ny = cp.info.ny, nz = cp.info.nz, nd = cp.adj_c1.n_os;
      std::string err;
      lfm_status st = k_transpose(w.z, w.zt, nz, ny, nd, nd, (long long)nz * nd, (long long)nd * ny, ny, stream, err);
      if (st != LFM_OK) return fail(st, err);
      TRY(sep(cp.adj_a2, w.zt, target, 0, nz, acc, stream));
    } else {
      TRY(sep(cp.adj_c2, w.z, target, 0, cp.info.nz, acc, stream));
    }
  } else if (plen) {
    TRY(sep(cp.adj_s3, y, w.f, 0, cp.info.n_views, 0, stream, 0, -1, r0, r1));
    TRY(sep(cp.adj_s1, w.f, target, 0, cp.info.nz, acc, stream));
  } else {
    TRY(sep(cp.adj_s1, y, target, 0, cp.info.nz, acc, stream, 0, -1, r0, r1));
  }
  if (rot) TRY(rotate_adj(cp, w.r0, x, accumulate, w, stream));
  return LFM_OK;
}

lfm_status check_path(int path) {
  if (path != LFM_PATH_PER_VIEW && path != LFM_PATH_COLLAPSED) return fail(LFM_E_INVALID, "unknown path");
  return LFM_OK;
}

}  // namespace

extern "C" {

const char* lfm_last_error(void) { return g_err.c_str(); }
const char* lfm_version(void) { return "liblfm 0.1 (sm_100a)"; }
int lfm_last_launch_count(void) { return g_last_launches; }

// View-subset forward / adjoint (per-view path over the subset's ops, then rotation as usual).
// A tensor-product subset (ViewOps::collapsed) runs on the collapsed two-pass path: band_v with the subset's s
// composite (K/|S| included), then the camera's full t pass; otherwise the per-view ops of the subset.
static bool subset_collapsed(const CameraPlan& cp, const ViewOps& vo) {
  return vo.collapsed && vo.vf.d_img && vo.va.d_img && cp.fwd_split && cp.fwd_t == 3 && cp.adj_t == 3;
}

lfm_status forward_subset_impl(const CameraPlan& cp, int m, const float* x, float* y, const Ws& w, void* stream) {
  const ViewOps& vo = cp.subs[m];
  const float* xr;
  TRY(rotate_fwd(cp, x, nullptr, 0, w, stream, &xr));
  if (subset_collapsed(cp, vo)) {
    bool amax_done = false;
    return vt_forward(cp, vo.vf, cp.fwd_c2, xr, y, 0, w, stream, Win(), amax_done);
  }
  if (cp.info.type == LFM_PLENOPTIC) {
    TRY(sep(vo.fwd_s1, xr, w.f, 0, vo.n_views, 0, stream));
    return sep(vo.fwd_s3, w.f, y, 0, 1, 0, stream);
  }
  return sep(vo.fwd_s1, xr, y, 0, 1, 0, stream);
}

lfm_status adjoint_subset_impl(const CameraPlan& cp, int m, const float* y, float* x, int accumulate, const Ws& w,
                               void* stream) {
  const ViewOps& vo = cp.subs[m];
  const bool rot = cp.info.rot_passes != 0;
  float* target = rot ? w.r0 : x;
  const int acc = rot ? 0 : accumulate;
  if (subset_collapsed(cp, vo)) {
    int split_state = 0;
    const bool z16 = z16_ok(cp, cp.adj_c1, vo.va);
    TRY(t_adjoint(cp, cp.adj_c1, y, w, stream, Win(), split_state, z16));
    std::string err;
    lfm_status st = k_vpass_adj(cp, vo.va, w.z, target, acc, stream, err, 0, -1, z16 ? w.am : nullptr,
                                cp.adj_c1.ft->u_lsum);
    if (st != LFM_OK) return fail(st, err);
  } else if (cp.info.type == LFM_PLENOPTIC) {
    TRY(sep(vo.adj_s3, y, w.f, 0, vo.n_views, 0, stream));
    TRY(sep(vo.adj_s1, w.f, target, 0, cp.info.nz, acc, stream));
  } else {
    TRY(sep(vo.adj_s1, y, target, 0, cp.info.nz, acc, stream));
  }
  if (rot) TRY(rotate_adj(cp, w.r0, x, accumulate, w, stream));
  return LFM_OK;
}

lfm_status lfm_plan_create(const lfm_geometry* g, int cuda_device, lfm_plan* out) {
  if (!out) return fail(LFM_E_INVALID, "out is NULL");
  *out = nullptr;
  if (!g || g->n_cam <= 0 || !g->cam) return fail(LFM_E_INVALID, "geometry has no cameras");
  lfm_plan_s* p = new lfm_plan_s;
  p->device = cuda_device;
  p->vol = g->vol;
  p->n_subsets = g->n_subsets > 1 ? g->n_subsets : 0;
  p->cams.resize(g->n_cam);
  for (int c = 0; c < g->n_cam; ++c) {
    std::string err;
    lfm_status st = build_camera(g->vol, g->cam[c], g->n_subsets, p->cams[c], err);
    if (st != LFM_OK) {
      delete p;
      return fail(st, "camera " + std::to_string(c) + ": " + err);
    }
  }
  WsLayout L = layout(p);
  for (CameraPlan& c : p->cams) c.info.ws_bytes = L.total;
  if (cuda_device >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    std::string err;
    lfm_status st = cuda_check(cudaSetDevice(cuda_device), "cudaSetDevice", err);
    for (int c = 0; st == LFM_OK && c < g->n_cam; ++c) {
      st = upload_camera(p->cams[c], err);
      if (st == LFM_OK) st = autotune_camera(p->cams[c], err);
      if (st == LFM_OK) st = prepare_subsets(p->cams[c], err);
      if (st != LFM_OK) err = "camera " + std::to_string(c) + ": " + err;
    }
    cudaSetDevice(prev);
    if (st != LFM_OK) {
      for (CameraPlan& c : p->cams) free_camera(c);
      delete p;
      return fail(st, err);
    }
  }
  *out = p;
  return LFM_OK;
}

lfm_status lfm_plan_destroy(lfm_plan p) {
  if (!p) return LFM_OK;
  if (p->device >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    for (CameraPlan& c : p->cams) free_camera(c);
    cudaSetDevice(prev);
  }
  delete p;
  return LFM_OK;
}

lfm_status lfm_plan_info(lfm_plan p, int cam, lfm_info* out) {
  lfm_status st = check_cam(p, cam, false);
  if (st != LFM_OK) return st;
  if (!out) return fail(LFM_E_INVALID, "out is NULL");
  *out = p->cams[cam].info;
  out->kind_stage[0] = p->cams[cam].fwd_c2.kind;
  out->kind_stage[1] = p->cams[cam].adj_c1.kind;
  out->subset_collapsed = 0;
  out->f16_stage[0] = p->device >= 0 && f16_fwd(p->cams[cam], p->cams[cam].fwd_c2) ? 1 : 0;
  out->f16_stage[1] = p->device >= 0 && f16_adj(p->cams[cam], p->cams[cam].adj_c1) ? 1 : 0;
  if (p->device >= 0)
    for (const ViewOps& vo : p->cams[cam].subs) out->subset_collapsed += subset_collapsed(p->cams[cam], vo) ? 1 : 0;
  return LFM_OK;
}

lfm_status lfm_plan_export_table(lfm_plan p, int cam, int table_id, int axis, int index, void* host_dst,
                                 size_t bytes, size_t* bytes_needed) {
  lfm_status st = check_cam(p, cam, false);
  if (st != LFM_OK) return st;
  const CameraPlan& cp = p->cams[cam];
  const void* srcp = nullptr;
  size_t need = 0;
  std::vector<char> tmp;
  if (table_id == LFM_TAB_SCALARS) {
    srcp = cp.scal;
    need = sizeof(cp.scal);
  } else if (table_id == LFM_TAB_ROT_MLO || table_id == LFM_TAB_ROT_W64) {
    if (index < 0 || index > 2) return fail(LFM_E_INVALID, "shear pass index must be 0 (z), 1 (x), 2 (y)");
    const ShearPass& sp = cp.rot[index];
    if (!sp.active) {
      need = 0;
    } else if (table_id == LFM_TAB_ROT_MLO) {
      srcp = sp.mlo[0].data();
      need = sp.mlo[0].size() * 4;
    } else {
      srcp = sp.w64[0].data();
      need = sp.w64[0].size() * 8;
    }
  } else {
    if (axis < 0 || axis > 1) return fail(LFM_E_INVALID, "axis must be 0 (s) or 1 (t)");
    const BandFamily* f = nullptr;
    int group = table_id / 3, kind = table_id % 3;
    switch (group) {
      case 0: f = &cp.s1f[axis]; break;
      case 1: f = &cp.s1a[axis]; break;
      case 2: f = &cp.s3f[axis]; break;
      case 3: f = &cp.s3a[axis]; break;
      case 4: f = &cp.cf[axis]; break;
      default: return fail(LFM_E_INVALID, "unknown table id");
    }
    if (index < 0 || index >= f->n_tables) return fail(LFM_E_INVALID, "table index out of range");
    size_t r0 = (size_t)index * f->n_rows;
    if (kind == 0) { srcp = f->start.data() + r0; need = (size_t)f->n_rows * 4; }
    else if (kind == 1) { srcp = f->len.data() + r0; need = (size_t)f->n_rows * 4; }
    else { srcp = f->w64.data() + r0 * f->taps; need = (size_t)f->n_rows * f->taps * 8; }
  }
  if (bytes_needed) *bytes_needed = need;
  if (!host_dst) return LFM_OK;
  if (bytes != need) return fail(LFM_E_INVALID, "export size mismatch: need " + std::to_string(need));
  if (need) std::memcpy(host_dst, srcp, need);
  return LFM_OK;
}

lfm_status lfm_lf_transport(lfm_plan p, int cam, int dst_plane, int src_plane, const float* src, float* dst,
                            void* ws, size_t ws_bytes, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  if (!src || !dst) return fail(LFM_E_INVALID, "src/dst is NULL");
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  const CameraPlan& cp = p->cams[cam];
  const int nz = cp.info.nz, K = cp.info.n_views;
  const bool plen = cp.info.type == LFM_PLENOPTIC;
  const int A = nz, D = nz + 1;
  auto is_slice = [&](int q) { return q >= 0 && q < nz; };
  if (plen) {
    if (dst_plane == A && is_slice(src_plane)) st = sep(cp.xp_s1f, src, dst, src_plane * K, K, 0, stream);
    else if (is_slice(dst_plane) && src_plane == A) st = sep(cp.xp_s1a, src, dst, dst_plane * K, K, 0, stream);
    else if (dst_plane == D && src_plane == A) st = sep(cp.xp_s3f, src, dst, 0, K, 0, stream);
    else if (dst_plane == A && src_plane == D) st = sep(cp.xp_s3a, src, dst, 0, K, 0, stream);
    else return fail(LFM_E_MISMATCH, "unsupported plane pair for a plenoptic camera");
  } else {
    if (dst_plane == D && is_slice(src_plane)) st = sep(cp.xp_s1f, src, dst, src_plane * K, K, 0, stream);
    else if (is_slice(dst_plane) && src_plane == D) st = sep(cp.xp_s1a, src, dst, dst_plane * K, K, 0, stream);
    else return fail(LFM_E_MISMATCH, "unsupported plane pair for a single-lens camera");
  }
  g_last_launches = g_launches;
  return st;
}

lfm_status lfm_vol_accumulate(const float* src, float* dst, long long n, void* stream) {
  g_launches = 0;
  if (n < 0) return fail(LFM_E_INVALID, "n < 0");
  if (n == 0) return LFM_OK;
  if (!src || !dst || src == dst) return fail(LFM_E_INVALID, "src/dst NULL or aliased");
  std::string err;
  lfm_status st = k_copy_scale(src, dst, n, 1.f, 1, stream, err);
  g_last_launches = g_launches;
  return st == LFM_OK ? st : fail(st, err);
}

lfm_status lfm_vol_rotate(lfm_plan p, int cam, int dir, const float* in, float* out, int accumulate, void* ws,
                          size_t ws_bytes, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  if (!in || !out || in == out) return fail(LFM_E_INVALID, "in/out NULL or aliased");
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  const CameraPlan& cp = p->cams[cam];
  if (dir == LFM_FWD) {
    const float* xr;
    st = rotate_fwd(cp, in, out, accumulate, w, stream, &xr);
  } else if (dir == LFM_ADJ) {
    st = rotate_adj(cp, in, out, accumulate, w, stream);
  } else {
    return fail(LFM_E_INVALID, "dir must be LFM_FWD or LFM_ADJ");
  }
  g_last_launches = g_launches;
  return st;
}

static lfm_status check_window(const lfm_plan_s* p, int cam, int row0, int row1, int col0, int col1) {
  const lfm_info& inf = p->cams[cam].info;
  if (row0 < 0 || row1 > inf.n_t || row0 >= row1) return fail(LFM_E_INVALID, "bad detector row range");
  if (col0 < 0 || col1 > inf.n_s || col0 >= col1) return fail(LFM_E_INVALID, "bad detector column range");
  return LFM_OK;
}

lfm_status lfm_A_forward_window(lfm_plan p, int cam, int path, int row0, int row1, int col0, int col1, const float* x,
                                float* y, void* ws, size_t ws_bytes, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  if ((st = check_path(path)) != LFM_OK) return st;
  if (!x || !y) return fail(LFM_E_INVALID, "x/y is NULL");
  if ((st = check_window(p, cam, row0, row1, col0, col1)) != LFM_OK) return st;
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  Win win;
  win.r0 = row0; win.r1 = row1; win.c0 = col0; win.c1 = col1;
  st = forward_impl(p->cams[cam], path, x, y, w, stream, win);
  g_last_launches = g_launches;
  return st;
}

lfm_status lfm_A_forward_rows(lfm_plan p, int cam, int path, int row0, int row1, const float* x, float* y,
                              void* ws, size_t ws_bytes, void* stream) {
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  return lfm_A_forward_window(p, cam, path, row0, row1, 0, p->cams[cam].info.n_s, x, y, ws, ws_bytes, stream);
}

lfm_status lfm_A_stage(lfm_plan p, int cam, int stage, const float* in, float* out, void* ws, size_t ws_bytes,
                       void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  const CameraPlan& cp = p->cams[cam];
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  if (stage == LFM_STAGE_FWD_T) {
    if (!cp.fwd_split) return fail(LFM_E_INVALID, "collapsed forward of this camera is not in two-pass form");
    if (!out) return fail(LFM_E_INVALID, "out is NULL");
    // as in A_forward, on the U (and, 2xFP16, its fp16 split and the maxima of x^r) the last forward or FWD_S left
    F16Src h;
    if (f16_fwd(cp, cp.fwd_c2)) {
      h.hi = reinterpret_cast<const uint16_t*>(w.z);
      h.lo = h.hi + (size_t)cp.cf[0].n_rows * cp.info.nz * cp.info.ny;
      h.amax = w.am;
      h.amax_scale = cp.vf.lsum;
    }
    st = sep(cp.fwd_c2, w.z, out, 0, 1, 0, stream, 0, -1, 0, -1, 0, -1, w.zt, cp.ws_z, h);
  } else if (stage == LFM_STAGE_ADJ_T) {
    if (!in) return fail(LFM_E_INVALID, "in is NULL");
    int split_state = 0;  // 2xFP16: includes the split of `in` (part of the t pass's cost); Z in fp16
    st = t_adjoint(cp, cp.adj_c1, in, w, stream, Win(), split_state, z16_ok(cp, cp.adj_c1, cp.va));
  } else if (stage == LFM_STAGE_FWD_S || stage == LFM_STAGE_ADJ_S) {
    const bool fwd = stage == LFM_STAGE_FWD_S;
    if (fwd ? !in : !out) return fail(LFM_E_INVALID, fwd ? "in is NULL" : "out is NULL");
    if (fwd ? !(cp.fwd_split && (cp.fwd_t == 2 || cp.fwd_t == 3)) : !(cp.adj_t == 2 || cp.adj_t == 3))
      return fail(LFM_E_INVALID, "the s pass of this camera is not a direct (band_v / spass) kernel");
    std::string err;
    if (fwd && cp.fwd_t == 3) {  // as in A_forward (2xFP16: maxima and split of `in`, U as fp16 hi / lo)
      if (f16_fwd(cp, cp.fwd_c2)) {
        uint16_t* x16 = cp.vf.d_h16 && cp.vf.BK == 32 && cp.info.nx % 8 == 0 ? reinterpret_cast<uint16_t*>(w.xt) : nullptr;
        st = x16 ? k_split16_rows(in, cp.info.ny * cp.info.nz, cp.info.nx, w.am, w.rs, x16, x16 + cp.info.n_vox, stream, err)
                 : k_amax(in, cp.info.n_vox, w.am, stream, err);
        if (st == LFM_OK) st = k_vpass_fwd(cp, cp.vf, in, w.z, stream, err, 0, -1, w.am, x16, w.rs);
      } else {
        st = k_vpass_fwd(cp, cp.vf, in, w.z, stream, err);
      }
    } else if (fwd) {
      st = k_spass_fwd(cp, in, w.z, stream, err);
    } else {  // on the Z (fp16 when the t pass wrote it so) and maxima the last ADJ_T / adjoint left
      const bool z16 = z16_ok(cp, cp.adj_c1, cp.va);
      st = cp.adj_t == 3 ? k_vpass_adj(cp, cp.va, w.z, out, 0, stream, err, 0, -1, z16 ? w.am : nullptr, cp.adj_c1.ft->u_lsum)
                         : k_spass_adj(cp, w.z, out, 0, stream, err);
    }
    if (st != LFM_OK) return fail(st, err);
  } else {
    return fail(LFM_E_INVALID, "unknown stage");
  }
  g_last_launches = g_launches;
  return st;
}

static lfm_status check_subset(lfm_plan p, int cam, int subset) {
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  if (subset < 0 || subset >= (int)p->cams[cam].subs.size())
    return fail(LFM_E_INVALID, "subset index outside the plan's n_subsets");
  return LFM_OK;
}

lfm_status lfm_A_forward_subset(lfm_plan p, int cam, int subset, const float* x, float* y, void* ws, size_t ws_bytes,
                                void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  lfm_status st = check_subset(p, cam, subset);
  if (st != LFM_OK) return st;
  if (!x || !y) return fail(LFM_E_INVALID, "x/y is NULL");
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  st = forward_subset_impl(p->cams[cam], subset, x, y, w, stream);
  g_last_launches = g_launches;
  return st;
}

lfm_status lfm_A_adjoint_subset(lfm_plan p, int cam, int subset, const float* y, float* x, int accumulate, void* ws,
                                size_t ws_bytes, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  lfm_status st = check_subset(p, cam, subset);
  if (st != LFM_OK) return st;
  if (!x || !y) return fail(LFM_E_INVALID, "x/y is NULL");
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  st = adjoint_subset_impl(p->cams[cam], subset, y, x, accumulate, w, stream);
  g_last_launches = g_launches;
  return st;
}

lfm_status lfm_A_forward(lfm_plan p, int cam, int path, const float* x, float* y, void* ws, size_t ws_bytes,
                         void* stream) {
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  return lfm_A_forward_rows(p, cam, path, 0, p->cams[cam].info.n_t, x, y, ws, ws_bytes, stream);
}

lfm_status lfm_A_adjoint_window(lfm_plan p, int cam, int path, int row0, int row1, int col0, int col1, const float* y,
                                float* x, int accumulate, void* ws, size_t ws_bytes, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  if ((st = check_path(path)) != LFM_OK) return st;
  if (!x || !y) return fail(LFM_E_INVALID, "x/y is NULL");
  if ((st = check_window(p, cam, row0, row1, col0, col1)) != LFM_OK) return st;
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  Win win;
  win.r0 = row0; win.r1 = row1; win.c0 = col0; win.c1 = col1;
  st = adjoint_impl(p->cams[cam], path, y, x, accumulate, w, stream, win);
  g_last_launches = g_launches;
  return st;
}

lfm_status lfm_A_adjoint_rows(lfm_plan p, int cam, int path, int row0, int row1, const float* y, float* x,
                              int accumulate, void* ws, size_t ws_bytes, void* stream) {
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  return lfm_A_adjoint_window(p, cam, path, row0, row1, 0, p->cams[cam].info.n_s, y, x, accumulate, ws, ws_bytes,
                              stream);
}

lfm_status lfm_A_adjoint(lfm_plan p, int cam, int path, const float* y, float* x, int accumulate, void* ws,
                         size_t ws_bytes, void* stream) {
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  return lfm_A_adjoint_rows(p, cam, path, 0, p->cams[cam].info.n_t, y, x, accumulate, ws, ws_bytes, stream);
}

lfm_status lfm_pwls_stats(lfm_plan p, int cam, const float* Ax, const float* y, const float* w_, double* stats3,
                          void* ws, size_t ws_bytes, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  lfm_status st = check_cam(p, cam);
  if (st != LFM_OK) return st;
  if (!Ax || !y || !w_ || !stats3) return fail(LFM_E_INVALID, "NULL argument");
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  std::string err;
  st = k_stats(Ax, y, w_, p->cams[cam].info.n_pix, w.p, stats3, stream, err);
  g_last_launches = g_launches;
  return st == LFM_OK ? st : fail(st, err);
}

lfm_status lfm_pwls_gains(lfm_plan p, const double* stats, double* gamma, int* flag, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  if (!p || p->device < 0) return fail(LFM_E_INVALID, "plan is NULL or host-only");
  if (!stats || !gamma) return fail(LFM_E_INVALID, "NULL argument");
  std::string err;
  lfm_status st = k_gains(stats, (int)p->cams.size(), gamma, flag, stream, err);
  g_last_launches = g_launches;
  return st == LFM_OK ? st : fail(st, err);
}

lfm_status lfm_pwls_grad(lfm_plan p, int path, int subset, int cam0, int cam1, const float* x, const float* const* y,
                         const float* const* wts, const float* const* Ax, const double* gamma, float beta, float nu,
                         int include_reg, float* grad, double* cost, void* ws, size_t ws_bytes, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  if (!p || p->device < 0) return fail(LFM_E_INVALID, "plan is NULL or host-only");
  if (cam0 < 0 || cam1 > (int)p->cams.size() || cam0 > cam1) return fail(LFM_E_INVALID, "bad camera range");
  if (!x || !grad || (cam1 > cam0 && (!y || !wts || !Ax || !gamma))) return fail(LFM_E_INVALID, "NULL argument");
  lfm_status st = subset < 0 ? check_path(path) : LFM_OK;
  if (st != LFM_OK) return st;
  if (subset >= 0 && subset >= p->n_subsets) return fail(LFM_E_INVALID, "subset index outside the plan's n_subsets");
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  std::string err;
  const long long nvox = (long long)p->vol.nx * p->vol.ny * p->vol.nz;
  const bool acc_in = (include_reg & LFM_GRAD_ACCUMULATE) != 0;  // grad holds a partial gradient: add to it
  if (acc_in && cost) return fail(LFM_E_INVALID, "LFM_GRAD_ACCUMULATE with a cost");
  include_reg &= 1;
  if (cam1 == cam0 && !acc_in) {
    if ((st = k_fill(grad, nvox, 0.f, stream, err)) != LFM_OK) return fail(st, err);
    if (cost) cudaMemsetAsync(cost, 0, sizeof(double), (cudaStream_t)stream);
  }
  for (int c = cam0; c < cam1; ++c) {
    const CameraPlan& cp = p->cams[c];
    if (!y[c] || !wts[c] || !Ax[c]) return fail(LFM_E_INVALID, "NULL per-camera pointer");
    if (!cost && subset < 0 && res_fusable(cp, path, Ax[c], y[c], wts[c])) {
      // r never stored: the adjoint's column-scaled input split computes it from Ax, y, w
      const ResSrc rs = {Ax[c], y[c], wts[c], gamma, c};
      if ((st = adjoint_impl(cp, path, nullptr, grad, acc_in || c > cam0, w, stream, Win(), &rs)) != LFM_OK) return st;
      continue;
    }
    st = k_residual(Ax[c], y[c], wts[c], gamma, c, w.s, cp.info.n_pix, w.p, cost, c > cam0, stream, err);
    if (st != LFM_OK) return fail(st, err);
    st = subset < 0 ? adjoint_impl(cp, path, w.s, grad, acc_in || c > cam0, w, stream)
                    : adjoint_subset_impl(cp, subset, w.s, grad, acc_in || c > cam0, w, stream);
    if (st != LFM_OK) return st;
  }
  if (include_reg) {
    st = k_reg26(x, grad, p->vol.nx, p->vol.ny, p->vol.nz, beta, nu, w.p, cost ? cost + 1 : nullptr, stream, err);
    if (st != LFM_OK) return fail(st, err);
  } else if (cost) {
    cudaMemsetAsync(cost + 1, 0, sizeof(double), (cudaStream_t)stream);
  }
  g_last_launches = g_launches;
  if (cuda_check(cudaGetLastError(), "pwls_grad", err) != LFM_OK) return fail(LFM_E_CUDA, err);
  // non-finite cost: when the cost is requested (and the stream is not being captured into a graph)
  // the call waits for it and checks both parts
  if (cost) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing((cudaStream_t)stream, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
      double h[2] = {0.0, 0.0};
      if (cuda_check(cudaMemcpyAsync(h, cost, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream), "cost copy", err) !=
              LFM_OK ||
          cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "cost sync", err) != LFM_OK)
        return fail(LFM_E_CUDA, err);
      if (!std::isfinite(h[0]) || !std::isfinite(h[1]))
        return fail(LFM_E_NONFINITE, "non-finite cost: data term " + std::to_string(h[0]) + ", prior term " +
                                         std::to_string(h[1]) + " (cameras " + std::to_string(cam0) + ".." +
                                         std::to_string(cam1 - 1) + ")");
    } else {
      cudaGetLastError();
    }
  }
  return LFM_OK;
}

lfm_status lfm_majoriser(lfm_plan p, int path, int cam0, int cam1, const float* const* wts, float beta, int mode,
                         float* d, void* ws, size_t ws_bytes, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  if (!p || p->device < 0) return fail(LFM_E_INVALID, "plan is NULL or host-only");
  if (cam0 < 0 || cam1 > (int)p->cams.size() || cam0 > cam1) return fail(LFM_E_INVALID, "bad camera range");
  if (!d || ((mode & LFM_MAJ_SUM) && cam1 > cam0 && !wts)) return fail(LFM_E_INVALID, "NULL argument");
  lfm_status st = check_path(path);
  if (st != LFM_OK) return st;
  Ws w;
  if ((st = get_ws(p, ws, ws_bytes, w)) != LFM_OK) return st;
  std::string err;
  const long long nvox = (long long)p->vol.nx * p->vol.ny * p->vol.nz;
  if (mode & LFM_MAJ_SUM) {
    if (cam1 == cam0 && (st = k_fill(d, nvox, 0.f, stream, err)) != LFM_OK) return fail(st, err);
    for (int c = cam0; c < cam1; ++c) {
      const CameraPlan& cp = p->cams[c];
      if (!wts[c]) return fail(LFM_E_INVALID, "NULL weight pointer");
      if ((st = k_fill(w.s, nvox, 1.f, stream, err)) != LFM_OK) return fail(st, err);
      if ((st = forward_impl(cp, path, w.s, w.s2, w, stream)) != LFM_OK) return st;
      if ((st = k_mul(w.s2, wts[c], w.s2, cp.info.n_pix, stream, err)) != LFM_OK) return fail(st, err);
      if ((st = adjoint_impl(cp, path, w.s2, d, c > cam0, w, stream)) != LFM_OK) return st;
    }
  }
  if (mode & LFM_MAJ_FINISH) {
    if ((st = k_majoriser_finish(d, nvox, 36.f * beta, stream, err)) != LFM_OK) return fail(st, err);
  }
  g_last_launches = g_launches;
  return LFM_OK;
}

lfm_status lfm_fista_update(lfm_plan p, float* x, float* z, const float* grad, const float* d, double t_old,
                            double t_new, void* stream) {
  DevGuard dev_guard(p);
  g_launches = 0;
  if (!p || p->device < 0) return fail(LFM_E_INVALID, "plan is NULL or host-only");
  if (!x || !z || !grad || !d) return fail(LFM_E_INVALID, "NULL argument");
  if (!(t_new > 0)) return fail(LFM_E_INVALID, "t_new must be > 0");
  std::string err;
  const long long nvox = (long long)p->vol.nx * p->vol.ny * p->vol.nz;
  lfm_status st = k_fista(x, z, grad, d, nvox, (float)((t_old - 1.0) / t_new), stream, err);
  g_last_launches = g_launches;
  return st == LFM_OK ? st : fail(st, err);
}

}  // extern "C"
