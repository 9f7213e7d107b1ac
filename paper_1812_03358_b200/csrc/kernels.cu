// liblfm CUDA kernels for sm_100a.
//
// sep_kernel: the paper's separable light-transport filter (eqn,xport,sep P:904-910)
//   summed over a list of terms:  out[b] = out_scale * sum_e scale_e (B_s[e] (x) B_t[e]) src_e.
//   Per term the CTA (one output tile) stages the source footprint of its tile in shared memory
//   (coalesced along s), filters along t first ("minor direction") into a second smem tile,
//   then filters along s from that tile into registers.  One thread owns each output element
//   (one-writer rule): no atomics, bitwise-deterministic.  Weights come from fp32 band
//   tables built in fp64 by plan.cpp; threads of a warp share a t-row (identical weights, no
//   divergent integral branches) and run along s (coalesced loads/stores).
// shear_kernel: one pass of the three-pass rotation (eqn,rot,toeplitz P:1186-1198).
// PWLS kernels: deterministic fp64 two-level reductions, residual, 26-neighbour regulariser,
//   FISTA update (eqn,pls P:299-317, Appendix A).
#include <cuda_pipeline.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lfm_internal.h"
#include "band_u.cuh"
#include "band_v.cuh"
#include "spass.cuh"
#include "lfm_kernels.h"

namespace lfm {

thread_local int g_launches = 0;
static int g_num_sms();
// Kernel attributes (dynamic shared memory limits) belong to a device context: one-time flags are kept per device.
constexpr int LFM_MAX_DEV = 64;
static int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < LFM_MAX_DEV) ? d : 0;
}

lfm_status cuda_check(cudaError_t e, const char* what, std::string& err) {
  if (e == cudaSuccess) return LFM_OK;
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return LFM_E_CUDA;
}

template <typename T>
static lfm_status dev_upload(T** dst, const void* src, size_t bytes, std::string& err) {
  *dst = nullptr;
  if (bytes == 0) return LFM_OK;
  cudaError_t e = cudaMalloc((void**)dst, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    err = "cudaMalloc of plan tables failed";
    return LFM_E_NOMEM;
  }
  return cuda_check(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "upload", err);
}

// tf32 value of an fp32 (round to nearest, ties away, low 13 bits cleared), as cvt.rna.tf32.f32
static float tf32_host(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u += 0x1000u;
  u &= 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

static lfm_status upload_family(BandFamily& f, size_t& bytes, std::string& err) {
  if (f.n_tables == 0) return LFM_OK;
  // device ELL layout [table][entry][pitch] with pitch = rows rounded up to 4 (16-byte cp.async rows)
  const int pitch = (f.n_rows + 3) / 4 * 4;
  const size_t per_h = (size_t)f.ell * f.n_rows, per_d = (size_t)f.ell * pitch;
  std::vector<float> w32((size_t)f.n_tables * per_d, 0.f);
  std::vector<int32_t> ix((size_t)f.n_tables * per_d, 0), cn((size_t)f.n_tables * pitch, 0);
  for (int m = 0; m < f.n_tables; ++m) {
    for (int r = 0; r < f.n_rows; ++r) cn[(size_t)m * pitch + r] = f.cnt[(size_t)m * f.n_rows + r];
    for (int k = 0; k < f.ell; ++k)
      for (int r = 0; r < f.n_rows; ++r) {
        w32[m * per_d + (size_t)k * pitch + r] = (float)f.ew64[m * per_h + (size_t)k * f.n_rows + r];  // one rounding
        ix[m * per_d + (size_t)k * pitch + r] = f.eidx[m * per_h + (size_t)k * f.n_rows + r];
      }
  }
  lfm_status st = dev_upload(&f.d_cnt, cn.data(), cn.size() * sizeof(int32_t), err);
  if (st != LFM_OK) return st;
  if ((st = dev_upload(&f.d_idx, ix.data(), ix.size() * sizeof(int32_t), err)) != LFM_OK) return st;
  if ((st = dev_upload(&f.d_w, w32.data(), w32.size() * sizeof(float), err)) != LFM_OK) return st;
  std::vector<int32_t> g4((size_t)f.n_tables * f.n_groups * 8);  // two int4 segments per group
  for (size_t i = 0; i < (size_t)f.n_tables * f.n_groups * 2; ++i) {
    g4[4 * i] = f.g_j0[i];
    g4[4 * i + 1] = f.g_w[i];
    g4[4 * i + 2] = f.g_off[i];
    g4[4 * i + 3] = 0;
  }
  std::vector<float> gw(f.g_w64.size() + 4);
  for (size_t i = 0; i < f.g_w64.size(); ++i) gw[i] = (float)f.g_w64[i];
  if ((st = dev_upload(&f.d_g, g4.data(), g4.size() * 4, err)) != LFM_OK) return st;
  bytes += cn.size() * 4 + ix.size() * 4 + w32.size() * 4 + g4.size() * 4 + gw.size() * 4;
  if (f.want_mseg) {
    std::vector<float> mw(f.m_w64.size() + 4);
    for (size_t i = 0; i < f.m_w64.size(); ++i) mw[i] = (float)f.m_w64[i];  // one rounding, like every table
    if ((st = dev_upload(&f.d_moff, f.m_off.data(), f.m_off.size() * 4, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_mseg, f.m_seg.data(), f.m_seg.size() * 4 + 16, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_mw, mw.data(), mw.size() * 4, err)) != LFM_OK) return st;
    bytes += f.m_off.size() * 4 + f.m_seg.size() * 4 + mw.size() * 4;
  }
  if (!f.f_off.empty()) {
    std::vector<float> fw(f.f_w64.size() + 16);
    for (size_t i = 0; i < f.f_w64.size(); ++i) fw[i] = (float)f.f_w64[i];
    std::vector<int32_t> fr(f.f_row);
    fr.resize(fr.size() + 8, 0);
    if ((st = dev_upload(&f.d_foff, f.f_off.data(), f.f_off.size() * 4, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_frow, fr.data(), fr.size() * 4, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_fw, fw.data(), fw.size() * 4, err)) != LFM_OK) return st;
    bytes += f.f_off.size() * 4 + fr.size() * 4 + fw.size() * 4;
  }

  if (!f.u_off.empty()) {
    std::vector<int32_t> uk(f.u_k0);
    uk.push_back(0);
    if ((st = dev_upload(&f.d_uoff, f.u_off.data(), f.u_off.size() * 4, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_uk0, uk.data(), uk.size() * 4, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_ua, f.u_a.data(), f.u_a.size() * 4, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_uh, f.u_h.data(), f.u_h.size() * 2, err)) != LFM_OK) return st;
    bytes += f.u_off.size() * 4 + uk.size() * 4 + f.u_a.size() * 4 + f.u_h.size() * 2;
  }
  if (!f.m8_off.empty()) {
    std::vector<float> mw(f.m8_w64.size() + 8);
    for (size_t i = 0; i < f.m8_w64.size(); ++i) mw[i] = (float)f.m8_w64[i];
    if ((st = dev_upload(&f.d_m8off, f.m8_off.data(), f.m8_off.size() * 4, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_m8seg, f.m8_seg.data(), f.m8_seg.size() * 4 + 16, err)) != LFM_OK) return st;
    if ((st = dev_upload(&f.d_m8w, mw.data(), mw.size() * 4, err)) != LFM_OK) return st;
    bytes += f.m8_off.size() * 4 + f.m8_seg.size() * 4 + mw.size() * 4;
  }
  return dev_upload(&f.d_gw, gw.data(), gw.size() * 4, err);
}

static lfm_status upload_sep(SepOp& op, size_t& bytes, std::string& err) {
  if (!op.fs) return LFM_OK;
  lfm_status st = dev_upload(&op.d_terms, op.terms.data(), op.terms.size() * sizeof(Term), err);
  if (st != LFM_OK) return st;
  st = dev_upload(&op.d_offs, op.offs.data(), op.offs.size() * sizeof(int32_t), err);
  if (st != LFM_OK) return st;
  const BandFamily& fs = *op.fs;
  const BandFamily& ft = *op.ft;
  op.ntx = (fs.n_rows + op.ts - 1) / op.ts;
  op.nty = (ft.n_rows + op.tt - 1) / op.tt;
  std::vector<TileT> vs((size_t)fs.n_tables * op.ntx), vt((size_t)ft.n_tables * op.nty);
  for (int m = 0; m < fs.n_tables; ++m)
    for (int x = 0; x < op.ntx; ++x) {
      int lo, w, wo, wl;
      g4_tile(fs, m, op.ts, x, lo, w, wo, wl);
      vs[(size_t)m * op.ntx + x] = TileT{lo, w, wo, wl};
    }
  for (int m = 0; m < ft.n_tables; ++m)
    for (int y = 0; y < op.nty; ++y) {
      int lo, w, wo, wl;
      g4_tile(ft, m, op.tt, y, lo, w, wo, wl);
      vt[(size_t)m * op.nty + y] = TileT{lo, w, wo, wl};
    }
  st = dev_upload(&op.d_fp_s, vs.data(), vs.size() * sizeof(TileT), err);
  if (st != LFM_OK) return st;
  bytes += op.terms.size() * sizeof(Term) + (vs.size() + vt.size()) * sizeof(TileT);

  return dev_upload(&op.d_fp_t, vt.data(), vt.size() * sizeof(TileT), err);
}

static void dfree(void* p) {
  if (p) cudaFree(p);
}

// band_v tables of one s composite (forward family f: rows = detector columns, K = vx; adjoint family a: rows = vx,
// K = s).  Weights rounded once to fp32, then split hi = rn_tf32(w), lo = rn_tf32(w - hi); image element (row r, k)
// at byte r*64 + k*4, bits [4,6) ^= [7,9) (64-byte swizzle) or r*128 + k*4 with bits [4,7) ^= [7,10) (128-byte).
static void build_vtab(const BandFamily& f, int N, int BK, VTab& T) {
  T.N = N;
  T.BK = BK;
  T.n_nt = (f.n_rows + N - 1) / N;
  T.off.assign((size_t)f.n_tables * T.n_nt + 1, 0);
  T.k0.clear();
  T.img.clear();
  double lsum = 0;
  for (size_t idx = 0; idx < (size_t)f.n_tables * f.n_rows; ++idx) {
    double r = 0;
    for (int e = 0; e < f.len[idx]; ++e) r += std::fabs((double)(float)f.w64[idx * f.taps + e]);
    lsum = std::max(lsum, r);
  }
  T.lsum = (float)(lsum * (1.0 + 1e-6));
  std::vector<float> raw;  // the fp32 weights in the hi image's positions (source of the fp16 split)
  std::vector<char> any(f.n_src + 32);
  const uint32_t smask = BK >= 32 ? 7u : 3u;  // Swizzle<3,4,3> (128 B) or Swizzle<2,4,3> (64 B)
  for (int m = 0; m < f.n_tables; ++m)
    for (int t = 0; t < T.n_nt; ++t) {
      T.off[(size_t)m * T.n_nt + t] = (int)T.k0.size();
      std::fill(any.begin(), any.end(), 0);
      const int r0 = t * N, r1 = std::min(f.n_rows, r0 + N);
      for (int r = r0; r < r1; ++r) {
        const size_t idx = (size_t)m * f.n_rows + r;
        for (int e = 0; e < f.len[idx]; ++e)
          if (f.w64[idx * f.taps + e] != 0.0) any[f.start[idx] + e] = 1;
      }
      int last = -(1 << 30);
      for (int kn = 0; kn < f.n_src; ++kn) {
        if (!any[kn] || kn < last + BK) continue;
        const int k = kn & ~7;  // TMA: the innermost box coordinate must sit on a 16-byte boundary (fp16: 8 elements)
        last = k;
        T.k0.push_back(k);
        const size_t base = T.img.size();
        T.img.resize(base + (size_t)2 * BK * N, 0.f);
        raw.resize(base / 2 + (size_t)BK * N, 0.f);
        for (int r = r0; r < r1; ++r) {
          const size_t idx = (size_t)m * f.n_rows + r;
          for (int kk = 0; kk < BK; ++kk) {
            const int e = k + kk - f.start[idx];
            if (e < 0 || e >= f.len[idx]) continue;
            const float w = (float)f.w64[idx * f.taps + e];
            const float wh = tf32_host(w), wl = tf32_host(w - wh);
            const int sub = BK < 32 ? BK : 32, sj = kk / sub;  // sub-images of one swizzle-atom row each
            uint32_t o = (uint32_t)((r - r0) * sub * 4 + (kk % sub) * 4);
            o ^= ((o >> 7) & smask) << 4;
            const size_t so = (size_t)sj * N * sub;
            T.img[base + so + o / 4] = wh;
            T.img[base + (size_t)BK * N + so + o / 4] = wl;
            raw[base / 2 + so + o / 4] = w;
          }
        }
      }
    }
  T.off[(size_t)f.n_tables * T.n_nt] = (int)T.k0.size();
  // 2xFP16 images: the fp32 weights w (one rounding from fp64), 2^wexp w -> fp16 hi + lo in the same (row, k)
  // positions, BK-half rows: 64-byte rows with the 64-byte swizzle (BK 32) or 128-byte rows with the 128-byte
  // swizzle (BK 64)
  T.h16.clear();
  if (BK == 32 || BK == 64) {
    float wmax = 0.f;
    for (size_t i = 0; i < raw.size(); ++i) wmax = std::max(wmax, std::fabs(raw[i]));
    int ex = 0;
    if (wmax > 0.f) std::frexp((double)wmax * 1.01, &ex);
    T.wexp = wmax > 0.f ? 15 - ex : 0;
    const size_t nb = T.k0.size();
    T.h16.assign(nb * 2 * BK * N, 0);
    for (size_t b = 0; b < nb; ++b)
      for (int r = 0; r < N; ++r)
        for (int kk = 0; kk < BK; ++kk) {
          // fp32 image: sub-images of 32 columns, 128-byte rows, 128-byte swizzle
          uint32_t o32 = (uint32_t)(r * 128 + (kk % 32) * 4);
          o32 ^= ((o32 >> 7) & 7u) << 4;
          const float w = raw[b * BK * N + (size_t)(kk / 32) * N * 32 + o32 / 4];
          const float ws = (float)std::ldexp((double)w, T.wexp);
          const uint16_t wh = f2h_rn(ws), wl = f2h_rn(ws - h2f(wh));
          uint32_t o16 = (uint32_t)(r * BK * 2 + kk * 2);
          o16 ^= ((o16 >> 7) & (BK == 64 ? 7u : 3u)) << 4;
          T.h16[b * 2 * BK * N + o16 / 2] = wh;
          T.h16[b * 2 * BK * N + (size_t)BK * N + o16 / 2] = wl;
        }
  }
}

static void build_vtabs(const BandFamily& ff, const BandFamily& fa, VTab& vf, VTab& va) {
  const int bk_f = std::getenv("LFM_VBK_F") ? std::atoi(std::getenv("LFM_VBK_F")) : 32;
  // adjoint K blocks of 64 detector columns: with the 2xFP16 Z (fp16) that is 128-byte rows per TMA row, which
  // measured 45.1 -> 36.9 us per camera against 32 (LFM_VBK_A selects 16 / 32 / 64)
  const int bk_a = std::getenv("LFM_VBK_A") ? std::atoi(std::getenv("LFM_VBK_A")) : 64;
  build_vtab(ff, 256, bk_f == 16 ? 16 : 32, vf);
  const int vn_a = std::getenv("LFM_VN_A") ? std::atoi(std::getenv("LFM_VN_A")) : 16;
  build_vtab(fa, vn_a == 32 ? 32 : 16, bk_a == 16 ? 16 : bk_a == 64 ? 64 : 32, va);
  if (std::getenv("LFM_DEBUG"))
    for (const VTab* T : {&vf, &va}) {
      int mx = 0, mn = 1 << 30;
      for (size_t i = 0; i + 1 < T->off.size(); ++i) {
        mx = std::max(mx, T->off[i + 1] - T->off[i]);
        mn = std::min(mn, T->off[i + 1] - T->off[i]);
      }
      std::fprintf(stderr, "[lfm] band_v N %d: items %zu blocks %zu (min %d max %d per item)\n", T->N,
                   T->off.size() - 1, T->k0.size(), mn, mx);
    }
}

static lfm_status upload_vtab(VTab& T, size_t& bytes, std::string& err) {
  lfm_status st;
  std::vector<int32_t> k0(T.k0);
  k0.push_back(0);
  if ((st = dev_upload(&T.d_off, T.off.data(), T.off.size() * 4, err)) != LFM_OK) return st;
  if ((st = dev_upload(&T.d_k0, k0.data(), k0.size() * 4, err)) != LFM_OK) return st;
  if (!T.img.empty() && (st = dev_upload(&T.d_img, T.img.data(), T.img.size() * 4, err)) != LFM_OK) return st;
  if (!T.h16.empty() && (st = dev_upload(&T.d_h16, T.h16.data(), T.h16.size() * 2, err)) != LFM_OK) return st;
  bytes += T.off.size() * 4 + k0.size() * 4 + T.img.size() * 4 + T.h16.size() * 2;
  std::vector<float>().swap(T.img);  // host copies not needed after upload
  std::vector<uint16_t>().swap(T.h16);
  return LFM_OK;
}

static void free_vtab(VTab& T) {
  dfree(T.d_off); dfree(T.d_k0); dfree(T.d_img); dfree(T.d_h16);
  T.d_off = nullptr; T.d_k0 = nullptr; T.d_img = nullptr; T.d_h16 = nullptr;
}

lfm_status upload_camera(CameraPlan& cp, std::string& err) {
  size_t bytes = 0;
  lfm_status st;
  for (int ax = 0; ax < 2; ++ax) {
    BandFamily* fams[] = {&cp.s1f[ax], &cp.s1a[ax], &cp.s3f[ax], &cp.s3a[ax], &cp.cf[ax], &cp.ca[ax]};
    for (BandFamily* f : fams)
      if ((st = upload_family(*f, bytes, err)) != LFM_OK) return st;
  }
  for (BandFamily* f : {&cp.id_s, &cp.id_t, &cp.id_vt, &cp.ca1n, &cp.cf1n})
    if ((st = upload_family(*f, bytes, err)) != LFM_OK) return st;
  SepOp* ops[] = {&cp.fwd_s1, &cp.fwd_s3, &cp.adj_s3, &cp.adj_s1, &cp.fwd_c, &cp.adj_c1, &cp.adj_c2,
                  &cp.xp_s1f, &cp.xp_s1a, &cp.xp_s3f, &cp.xp_s3a, &cp.fwd_c1, &cp.fwd_c2, &cp.fwd_p1, &cp.adj_a2};
  for (SepOp* op : ops)
    if ((st = upload_sep(*op, bytes, err)) != LFM_OK) return st;
  for (int p = 0; p < 3; ++p) {
    ShearPass& sp = cp.rot[p];
    if (!sp.active) continue;
    for (int d = 0; d < 2; ++d) {
      std::vector<float> w32(sp.w64[d].size());
      for (size_t i = 0; i < w32.size(); ++i) w32[i] = (float)sp.w64[d][i];
      if ((st = dev_upload(&sp.d_mlo[d], sp.mlo[d].data(), sp.mlo[d].size() * 4, err)) != LFM_OK) return st;
      if ((st = dev_upload(&sp.d_w[d], w32.data(), w32.size() * 4, err)) != LFM_OK) return st;
      bytes += sp.mlo[d].size() * 4 + w32.size() * 4;
    }
  }
  // tcgen05 s passes (band_v.cuh): forward items (slice n, 256 detector columns), K = vx, from cf[0];
  // adjoint items (slice n, 16 voxel columns), K = s, from ca[0]
  build_vtabs(cp.cf[0], cp.ca[0], cp.vf, cp.va);
  for (VTab* T : {&cp.vf, &cp.va})
    if ((st = upload_vtab(*T, bytes, err)) != LFM_OK) return st;
  // terms >= 1 of a non-separable lenslet stage: t families (tcgen05 images), their ops, band_v tables
  for (Component& cm : cp.comps) {
    for (BandFamily* f : {&cm.ca1n, &cm.cf1n})
      if ((st = upload_family(*f, bytes, err)) != LFM_OK) return st;
    for (SepOp* op : {&cm.fwd_c2, &cm.adj_c1})
      if ((st = upload_sep(*op, bytes, err)) != LFM_OK) return st;
    build_vtabs(cm.cf[0], cm.ca[0], cm.vf, cm.va);
    for (VTab* T : {&cm.vf, &cm.va})
      if ((st = upload_vtab(*T, bytes, err)) != LFM_OK) return st;
  }
  cp.info.table_bytes = bytes;
  return LFM_OK;
}

lfm_status k_spass_fwd(const CameraPlan& cp, const float* x, float* U, void* stream, std::string& err) {
  const BandFamily& f = cp.cf[0];
  const int nx = cp.info.nx, ny = cp.info.ny, nz = cp.info.nz, nd = f.n_rows;
  const int pitch = (f.n_rows + 3) / 4 * 4;
  dim3 grid((nd + 255) / 256, nz, (ny + SPF_VTG - 1) / SPF_VTG);
  const size_t smem = (size_t)SPF_VTG * nx * 4;
  if (smem > 48 * 1024) { err = "spass_fwd: volume rows too long"; return LFM_E_INVALID; }
  spass_fwd_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(x, U, f.d_cnt, f.d_idx, f.d_w, nx, ny, nz, nd, f.ell, pitch);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "spass_fwd_kernel launch", err);
}

lfm_status k_spass_adj(const CameraPlan& cp, const float* Z, float* out, int accumulate, void* stream, std::string& err) {
  const BandFamily& f = cp.ca[0];
  const int nx = cp.info.nx, ny = cp.info.ny, nz = cp.info.nz, nd = cp.adj_c1.n_os;  // Z rows: detector columns
  const int pitch = (f.n_rows + 3) / 4 * 4;
  const int vta = std::getenv("LFM_SPA_VTA") ? (std::atoi(std::getenv("LFM_SPA_VTA")) == 4 ? 4 : 8) : (cp.spa_vta == 4 ? 4 : 8);
  const size_t smem = (size_t)vta * (nd + (nd >> 4) + 4) * 4;
  static size_t smem_set[LFM_MAX_DEV][2];
  size_t& ss0 = smem_set[cur_dev()][vta == 8];
  if (ss0 == 0) ss0 = 48 * 1024;
  size_t& ss = ss0;
  if (smem > ss) {
    cudaError_t e = vta == 8 ? cudaFuncSetAttribute(spass_adj_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                             : cudaFuncSetAttribute(spass_adj_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (smem > 200 * 1024 || e != cudaSuccess) {
      cudaGetLastError();
      err = "spass_adj: detector rows exceed shared memory";
      return LFM_E_INVALID;
    }
    ss = smem;
  }
  dim3 grid((ny + vta - 1) / vta, nz);
  if (vta == 8)
    spass_adj_kernel<8><<<grid, 128, smem, (cudaStream_t)stream>>>(Z, out, f.d_cnt, f.d_idx, f.d_w, nx, ny, nz, nd, f.ell,
                                                                  pitch, cp.adj_c2.out_scale, accumulate);
  else
    spass_adj_kernel<4><<<grid, 128, smem, (cudaStream_t)stream>>>(Z, out, f.d_cnt, f.d_idx, f.d_w, nx, ny, nz, nd, f.ell,
                                                                  pitch, cp.adj_c2.out_scale, accumulate);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "spass_adj_kernel launch", err);
}

// ---------------------------------------------------------------------------------------------- band_v host side
// Tensor-map cache (per host thread): the maps depend only on (base, dims, strides, box, swizzle), and the same
// buffers come back every call, so an apply call re-encodes nothing after its first use (host launch overhead).
struct TmapKey {
  const void* base;
  long long v[11];
};
struct TmapEntry {
  TmapKey key;
  CUtensorMap map;
};
static std::vector<TmapEntry>& tmap_cache() {
  thread_local std::vector<TmapEntry> cache;
  return cache;
}
static bool tmap_lookup(const TmapKey& k, CUtensorMap* out) {
  for (const TmapEntry& e : tmap_cache())
    if (e.key.base == k.base && std::memcmp(e.key.v, k.v, sizeof(k.v)) == 0) {
      *out = e.map;
      return true;
    }
  return false;
}
static void tmap_insert(const TmapKey& k, const CUtensorMap& m) {
  std::vector<TmapEntry>& c = tmap_cache();
  if (c.size() >= 64) c.erase(c.begin());  // bounded: oldest first
  c.push_back({k, m});
}

typedef CUresult (*EncodeTiledFnV)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static lfm_status encode3_raw(CUtensorMap* map, const void* base, const long long dims[3], const long long strides[2],
                          const int box[3], CUtensorMapSwizzle swz, std::string& err, bool f16 = false) {
  static EncodeTiledFnV encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &qr) != cudaSuccess || !encode) {
      cudaGetLastError();
      err = "band_v: cuTensorMapEncodeTiled unavailable";
      return LFM_E_CUDA;
    }
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (strides[0] & 15) || (strides[1] & 15)) {
    err = "band_v: buffers and their rows must be 16-byte aligned";
    return LFM_E_INVALID;
  }
  cuuint64_t gd[3] = {(cuuint64_t)dims[0], (cuuint64_t)dims[1], (cuuint64_t)dims[2]};
  cuuint64_t gs[2] = {(cuuint64_t)strides[0], (cuuint64_t)strides[1]};
  cuuint32_t bx[3] = {(cuuint32_t)box[0], (cuuint32_t)box[1], (cuuint32_t)box[2]}, es[3] = {1, 1, 1};
  CUresult r = encode(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), gd, gs, bx, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "band_v: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return LFM_E_CUDA;
  }
  return LFM_OK;
}

static lfm_status encode3(CUtensorMap* map, const void* base, const long long dims[3], const long long strides[2],
                          const int box[3], CUtensorMapSwizzle swz, std::string& err, bool f16 = false) {
  const TmapKey k = {base, {3, dims[0], dims[1], dims[2], strides[0], strides[1], box[0], box[1], box[2], (long long)swz, f16}};
  if (tmap_lookup(k, map)) return LFM_OK;
  lfm_status st = encode3_raw(map, base, dims, strides, box, swz, err, f16);
  if (st == LFM_OK) tmap_insert(k, *map);
  return st;
}

// 2D tensor map of a row-major matrix (rows x cols, pitch in elements; cached per host thread), defined below
static lfm_status encode_map(CUtensorMap* map, const void* base, int cols, int rows, long long pitch, int box_c,
                             int box_r, CUtensorMapSwizzle swz, std::string& err, bool f16 = false);

template <int N, int DIR, int BK, bool OUT16 = false, bool IN16 = false>
static lfm_status launch_band_v(const VTab& T, const CUtensorMap& am, const CUtensorMap& om, int nz, int ny,
                                float scale, int accumulate, void* stream, std::string& err, int nt0 = 0, int nt_cnt = -1,
                                int k_lo = 0, int k_hi = 1 << 30, const CUtensorMap* lom = nullptr,
                                const float* amax = nullptr, const CUtensorMap* alom = nullptr, float in_scale = 1.f,
                                const float* rinv = nullptr) {
  // the K-window instantiation only when a window cuts the K range (adjoint column shards)
  const bool kwin = k_lo > 0 || k_hi < (1 << 30);
  static bool attr[LFM_MAX_DEV][2];
  const int dv = cur_dev();
  constexpr size_t SMEM = VCfg<N, BK, IN16, OUT16>::SMEM;
  if (!attr[dv][kwin]) {
    cudaError_t e = kwin ? cudaFuncSetAttribute(band_v_kernel<N, DIR, BK, true, OUT16, IN16>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM)
                         : cudaFuncSetAttribute(band_v_kernel<N, DIR, BK, false, OUT16, IN16>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) return cuda_check(cudaGetLastError(), "band_v smem attribute", err);
    attr[dv][kwin] = true;
  }
  VArgs v;
  v.B = T.d_img;
  v.H = T.d_h16;
  v.blk_off = T.d_off;
  v.blk_k0 = T.d_k0;
  v.nz = nz;
  v.n_mt = (ny + 127) / 128;
  v.n_nt = T.n_nt;
  v.nt0 = std::max(0, nt0);
  v.nt_cnt = nt_cnt < 0 ? T.n_nt - v.nt0 : std::min(nt_cnt, T.n_nt - v.nt0);
  v.k_lo = kwin ? k_lo : 0;
  v.k_hi = k_hi;
  v.group = 4;
  v.scale = IN16 ? (float)std::ldexp((double)scale, -T.wexp) : scale;
  v.accumulate = accumulate;
  v.amax = amax;
  v.amax_scale = T.lsum;
  v.in_scale = in_scale;
  v.rinv = rinv;
  v.ny = ny;
  const int items = v.nz * v.n_mt * v.nt_cnt;
  if (items <= 0) return LFM_OK;
  const int grid = std::min(items, g_num_sms());
  const CUtensorMap& lm = lom ? *lom : om;
  const CUtensorMap& alm = alom ? *alom : am;
  if (kwin) band_v_kernel<N, DIR, BK, true, OUT16, IN16><<<grid, V_THREADS, SMEM, (cudaStream_t)stream>>>(am, om, lm, alm, v);
  else band_v_kernel<N, DIR, BK, false, OUT16, IN16><<<grid, V_THREADS, SMEM, (cudaStream_t)stream>>>(am, om, lm, alm, v);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "band_v_kernel launch", err);
}

lfm_status k_vpass_fwd(const CameraPlan& cp, const VTab& T, const float* x, float* U, void* stream, std::string& err,
                       int c0, int c1, const float* amax, const uint16_t* x16, const float* rinv) {
  const int nx = cp.info.nx, ny = cp.info.ny, nz = cp.info.nz, nd = cp.cf[0].n_rows;
  if (!T.d_img) { err = "band_v: no forward tables"; return LFM_E_INVALID; }
  CUtensorMap am, om;
  const int ob[3] = {32, 1, 32};
  const int ob16[3] = {64, 1, 32};  // fp16 U: 64-column boxes (VCfg O16)
  // column window [c0, c1): only the N-tiles (256 detector columns) that meet it
  const int nt0 = std::max(0, c0) / T.N, nt1 = c1 < 0 ? T.n_nt : (c1 + T.N - 1) / T.N;
  lfm_status st;
  if (amax && x16 && T.d_h16 && T.BK == 32) {  // 2xFP16 in and out: x^r pre-split (fp16 hi, lo = hi + n_vox)
    const long long ad[3] = {nx, ny, nz}, as[2] = {(long long)nx * 2, (long long)nx * ny * 2};
    const int ab[3] = {32, 128, 1};
    CUtensorMap alm, lm;
    const uint16_t* hi = reinterpret_cast<const uint16_t*>(U);
    const uint16_t* lo = hi + (size_t)nd * nz * ny;
    const long long od[3] = {nd, nz, ny}, os[2] = {(long long)nd * 2, (long long)nz * nd * 2};
    if ((st = encode3(&am, x16, ad, as, ab, CU_TENSOR_MAP_SWIZZLE_64B, err, true)) != LFM_OK ||
        (st = encode3(&alm, x16 + cp.info.n_vox, ad, as, ab, CU_TENSOR_MAP_SWIZZLE_64B, err, true)) != LFM_OK ||
        (st = encode3(&om, hi, od, os, ob16, CU_TENSOR_MAP_SWIZZLE_128B, err, true)) != LFM_OK ||
        (st = encode3(&lm, lo, od, os, ob16, CU_TENSOR_MAP_SWIZZLE_128B, err, true)) != LFM_OK)
      return st;
    return launch_band_v<256, 0, 32, true, true>(T, am, om, nz, ny, 1.f, 0, stream, err, nt0, nt1 - nt0, 0, 1 << 30, &lm,
                                                 amax, &alm, 1.f, rinv);
  }
  const long long ad[3] = {nx, ny, nz}, as[2] = {(long long)nx * 4, (long long)nx * ny * 4};
  const int ab[3] = {T.BK, 128, 1};
  st = encode3(&am, x, ad, as, ab, T.BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, err);
  if (st != LFM_OK) return st;
  if (amax) {  // fp16 hi / lo of 2^e U (the 2xFP16 t pass input): two [vt][n][s] half arrays
    const uint16_t* hi = reinterpret_cast<const uint16_t*>(U);
    const uint16_t* lo = hi + (size_t)nd * nz * ny;
    const long long od[3] = {nd, nz, ny}, os[2] = {(long long)nd * 2, (long long)nz * nd * 2};
    CUtensorMap lm;
    if ((st = encode3(&om, hi, od, os, ob, CU_TENSOR_MAP_SWIZZLE_64B, err, true)) != LFM_OK) return st;
    if ((st = encode3(&lm, lo, od, os, ob, CU_TENSOR_MAP_SWIZZLE_64B, err, true)) != LFM_OK) return st;
    return T.BK == 32 ? launch_band_v<256, 0, 32, true>(T, am, om, nz, ny, 1.f, 0, stream, err, nt0, nt1 - nt0, 0, 1 << 30, &lm, amax)
                      : launch_band_v<256, 0, 16, true>(T, am, om, nz, ny, 1.f, 0, stream, err, nt0, nt1 - nt0, 0, 1 << 30, &lm, amax);
  }
  const long long od[3] = {nd, nz, ny}, os[2] = {(long long)nd * 4, (long long)nz * nd * 4};
  if ((st = encode3(&om, U, od, os, ob, CU_TENSOR_MAP_SWIZZLE_128B, err)) != LFM_OK) return st;
  return T.BK == 32 ? launch_band_v<256, 0, 32>(T, am, om, nz, ny, 1.f, 0, stream, err, nt0, nt1 - nt0)
                    : launch_band_v<256, 0, 16>(T, am, om, nz, ny, 1.f, 0, stream, err, nt0, nt1 - nt0);
}

lfm_status k_vpass_adj(const CameraPlan& cp, const VTab& T, const float* Z, float* out, int accumulate, void* stream,
                       std::string& err, int c0, int c1, const float* amax, float in_scale) {
  const bool in16 = amax && vpass_adj_in16(T);
  const int nx = cp.info.nx, ny = cp.info.ny, nz = cp.info.nz, nd = cp.adj_c1.n_os;
  if (!T.d_img) { err = "band_v: no adjoint tables"; return LFM_E_INVALID; }
  // column window [c0, c1) of Z (= of y): the data map starts at c0 and is c1 - c0 wide, so columns outside read
  // as zeros; K blocks outside the window are skipped (items without live blocks write zeros)
  const int k_lo = std::max(0, c0), k_hi = (c1 < 0 || c1 >= nd) ? (1 << 30) : c1;
  if (k_lo % 4) { err = "band_v: a column window must start on a multiple of 4"; return LFM_E_INVALID; }
  CUtensorMap am, om, alm;
  lfm_status st;
  if (in16) {  // Z as fp16 hi (Z reinterpreted) and lo (the next nd nz ny halves) of 2^e Z
    const uint16_t* zh = reinterpret_cast<const uint16_t*>(Z);
    const uint16_t* zl = zh + (size_t)nd * nz * ny;
    const long long ad[3] = {std::min(k_hi, nd) - k_lo, nz, ny}, as[2] = {(long long)nd * 2, (long long)nz * nd * 2};
    const int ab[3] = {T.BK, 1, 128};
    const CUtensorMapSwizzle sw = T.BK == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    if ((st = encode3(&am, zh + k_lo, ad, as, ab, sw, err, true)) != LFM_OK ||
        (st = encode3(&alm, zl + k_lo, ad, as, ab, sw, err, true)) != LFM_OK)
      return st;
  } else {
    const long long ad[3] = {std::min(k_hi, nd) - k_lo, nz, ny}, as[2] = {(long long)nd * 4, (long long)nz * nd * 4};
    Z += k_lo;
    const int ab[3] = {T.BK < 32 ? T.BK : 32, 1, 128};
    st = encode3(&am, Z, ad, as, ab, T.BK >= 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, err);
    if (st != LFM_OK) return st;
  }
  const long long od[3] = {nx, ny, nz}, os[2] = {(long long)nx * 4, (long long)nx * ny * 4};
  const int ob[3] = {T.N / 2, 32, 1};
  if ((st = encode3(&om, out, od, os, ob, CU_TENSOR_MAP_SWIZZLE_NONE, err)) != LFM_OK) return st;
  const float sc = cp.adj_c2.out_scale;
  // a column window reaches only the voxel-column tiles whose K blocks meet it (host copy of the block starts):
  // launch those; the rest of the output is zero (memset first unless accumulating)
  int nt0 = 0, nt_cnt = -1;
  if (k_lo > 0 || k_hi < (1 << 30)) {
    int lo = T.n_nt, hi = -1;
    for (int nt = 0; nt < T.n_nt; ++nt)
      for (int n = 0; n < nz && !(lo <= nt && nt <= hi); ++n) {
        const size_t key = (size_t)n * T.n_nt + nt;
        for (int b = T.off[key]; b < T.off[key + 1]; ++b)
          if (T.k0[b] + T.BK > k_lo && T.k0[b] < k_hi) {
            lo = std::min(lo, nt);
            hi = std::max(hi, nt);
            break;
          }
      }
    nt0 = hi < 0 ? 0 : lo;
    nt_cnt = hi < 0 ? 0 : hi - lo + 1;
    if (!accumulate && (nt0 > 0 || nt0 + nt_cnt < T.n_nt)) {
      if (cudaMemsetAsync(out, 0, (size_t)nx * ny * nz * 4, (cudaStream_t)stream) != cudaSuccess)
        return cuda_check(cudaGetLastError(), "band_v window memset", err);
    }
    if (nt_cnt == 0) return LFM_OK;
  }
  if (in16)
    return T.BK == 64 ? launch_band_v<16, 1, 64, false, true>(T, am, om, nz, ny, sc, accumulate, stream, err, nt0, nt_cnt,
                                                              k_lo, k_hi, nullptr, amax, &alm, in_scale)
                      : launch_band_v<16, 1, 32, false, true>(T, am, om, nz, ny, sc, accumulate, stream, err, nt0, nt_cnt,
                                                              k_lo, k_hi, nullptr, amax, &alm, in_scale);
  if (T.N == 32)
    return T.BK == 32 ? launch_band_v<32, 1, 32>(T, am, om, nz, ny, sc, accumulate, stream, err, nt0, nt_cnt, k_lo, k_hi)
                      : launch_band_v<32, 1, 16>(T, am, om, nz, ny, sc, accumulate, stream, err, nt0, nt_cnt, k_lo, k_hi);
  if (T.BK == 64) return launch_band_v<16, 1, 64>(T, am, om, nz, ny, sc, accumulate, stream, err, nt0, nt_cnt, k_lo, k_hi);
  return T.BK == 32 ? launch_band_v<16, 1, 32>(T, am, om, nz, ny, sc, accumulate, stream, err, nt0, nt_cnt, k_lo, k_hi)
                    : launch_band_v<16, 1, 16>(T, am, om, nz, ny, sc, accumulate, stream, err, nt0, nt_cnt, k_lo, k_hi);
}

// Subset ops reuse the tile configuration the autotuner chose for the full per-view op (same tables,
// fewer terms per output, so the staged footprints and shared memory only shrink).
lfm_status prepare_subsets(CameraPlan& cp, std::string& err) {
  size_t bytes = 0;
  for (ViewOps& vo : cp.subs) {
    if (vo.collapsed) {
      build_vtabs(vo.cfs, vo.cas, vo.vf, vo.va);
      for (VTab* T : {&vo.vf, &vo.va}) {
        lfm_status st = upload_vtab(*T, bytes, err);
        if (st != LFM_OK) return st;
      }
    }
    SepOp* pairs[][2] = {{&vo.fwd_s1, &cp.fwd_s1}, {&vo.fwd_s3, &cp.fwd_s3}, {&vo.adj_s3, &cp.adj_s3},
                         {&vo.adj_s1, &cp.adj_s1}};
    for (auto& pr : pairs) {
      SepOp& op = *pr[0];
      const SepOp& full = *pr[1];
      if (!op.fs) continue;
      op.ts = full.ts; op.tt = full.tt; op.nt = full.nt; op.nb = full.nb; op.stage = full.stage;
      op.kind = full.kind; op.stages = full.stages; op.mgrp = full.mgrp; op.chunk = full.chunk;
      fill_sep_geometry(op);
      lfm_status st = upload_sep(op, bytes, err);
      if (st != LFM_OK) return st;
    }
  }
  return LFM_OK;
}

void free_camera(CameraPlan& cp) {
  for (VTab* T : {&cp.vf, &cp.va}) free_vtab(*T);
  for (ViewOps& vo : cp.subs) {
    free_vtab(vo.vf);
    free_vtab(vo.va);
  }
  for (Component& cm : cp.comps) {
    free_vtab(cm.vf);
    free_vtab(cm.va);
  }

  std::vector<BandFamily*> fams = {&cp.id_s, &cp.id_t, &cp.id_vt, &cp.ca1n, &cp.cf1n};
  for (Component& cm : cp.comps)
    for (BandFamily* f : {&cm.ca1n, &cm.cf1n}) fams.push_back(f);
  for (int ax = 0; ax < 2; ++ax)
    for (BandFamily* f : {&cp.s1f[ax], &cp.s1a[ax], &cp.s3f[ax], &cp.s3a[ax], &cp.cf[ax], &cp.ca[ax]})
      fams.push_back(f);
  for (BandFamily* f : fams) {
    dfree(f->d_cnt); dfree(f->d_idx); dfree(f->d_w); dfree(f->d_g); dfree(f->d_gw);
    dfree(f->d_moff); dfree(f->d_mseg); dfree(f->d_mw); dfree(f->d_m8off); dfree(f->d_m8seg); dfree(f->d_m8w);
    f->d_m8off = nullptr; f->d_m8seg = nullptr; f->d_m8w = nullptr;
    dfree(f->d_foff); dfree(f->d_frow); dfree(f->d_fw);
    f->d_foff = nullptr; f->d_frow = nullptr; f->d_fw = nullptr;
    dfree(f->d_uoff); dfree(f->d_uk0); dfree(f->d_ua); dfree(f->d_uh);
    f->d_uoff = nullptr; f->d_uk0 = nullptr; f->d_ua = nullptr; f->d_uh = nullptr;
    f->d_cnt = nullptr; f->d_idx = nullptr; f->d_w = nullptr; f->d_g = nullptr; f->d_gw = nullptr;
    f->d_moff = nullptr; f->d_mseg = nullptr; f->d_mw = nullptr;
  }
  SepOp* ops[] = {&cp.fwd_s1, &cp.fwd_s3, &cp.adj_s3, &cp.adj_s1, &cp.fwd_c, &cp.adj_c1, &cp.adj_c2,
                  &cp.xp_s1f, &cp.xp_s1a, &cp.xp_s3f, &cp.xp_s3a, &cp.fwd_c1, &cp.fwd_c2, &cp.fwd_p1, &cp.adj_a2};
  std::vector<SepOp*> all(std::begin(ops), std::end(ops));
  for (ViewOps& vo : cp.subs)
    for (SepOp* op : {&vo.fwd_s1, &vo.fwd_s3, &vo.adj_s3, &vo.adj_s1}) all.push_back(op);
  for (Component& cm : cp.comps)
    for (SepOp* op : {&cm.fwd_c2, &cm.adj_c1}) all.push_back(op);
  for (SepOp* op : all) {
    dfree(op->d_terms); dfree(op->d_offs); dfree(op->d_fp_s); dfree(op->d_fp_t);
    op->d_terms = nullptr; op->d_offs = nullptr; op->d_fp_s = nullptr; op->d_fp_t = nullptr;
  }
  for (int p = 0; p < 3; ++p)
    for (int d = 0; d < 2; ++d) {
      dfree(cp.rot[p].d_mlo[d]);
      dfree(cp.rot[p].d_w[d]);
      cp.rot[p].d_mlo[d] = nullptr;
      cp.rot[p].d_w[d] = nullptr;
    }
}

// ------------------------------------------------------------------------------------------
// Separable banded sum.  For every term (one slice / view / transport) of an output tile:
//   pass 1 (s direction): U[r][4g+q] = sum_p Ws_g[p][q] * X[r][j0_g + p]   (G4 s table: groups of 4
//          output columns share a window of source columns; one LDS.128 of weights feeds 4 FFMAs
//          per staged source row handled by the thread);
//   pass 2 (t direction, the large pass): out[4g+q][c] += sum_p Wt_g[p][q] * U[j0_g + p][c] with the
//          weights of a group of 4 output rows shared by the whole warp (broadcast) and 4 columns
//          per thread: one LDS.128 of weights + one LDS.128 of U feed 16 FFMAs.
// Chunks of nb terms (headers, source footprint, weights, group descriptors) are staged with cp.async
// into a double buffer, so the loads of chunk i+1 overlap the two passes of chunk i.  One thread owns
// each output element: no atomics; results are bitwise reproducible.
struct SepArgs {
  const float* src;
  float* out;
  long long out_stride;
  long long src_pitch;  // floats between source rows
  long long out_pitch;  // floats between output rows
  const int32_t* t_foff;  // flat MSEG entries (band_f_kernel)
  const int4* t_frow;
  const float4* t_fw;
  const int32_t* t_moff;  // MSEG t family (band_m_kernel)
  const int4* t_mseg;
  const float* t_mw;
  const Term* terms;
  const int32_t* offs;  // already offset by b0
  const int4* s_g;
  const float* s_gw;
  const int4* t_g;
  const float* t_gw;
  const TileT* fp_s;
  const TileT* fp_t;
  int s_ngroups, t_ngroups;
  int ntx, nty;
  int n_os, n_ot, n_is, n_it;
  int fsp, ftm, wsm, wtm, nb, nbuf;
  int s_ident;  // s table is the identity: pass 1 is a copy (source rows staged straight into U)
  int ug;       // identity s: pass 2 reads U rows straight from the source in global memory (no U tile)
  int ty0;      // first output t tile of this launch (detector-row sharding)
  int win_r0, win_r1;  // source rows outside [win_r0, win_r1) are treated as zero (adjoint row sharding)
  float out_scale;
  int accumulate;
};

struct SlotLayout {
  int xs, ws, gs, wt, gt, per;
};
// per staged term: [source footprint X (mode 0)] [s weights] [s group descriptors: 2 int4 per group]
// [t weights] [t group descriptors: 2 int4 per group]; must match sep_smem() in plan.cpp
__host__ __device__ inline SlotLayout slot_layout(int ftm, int fsp, bool xs, int wsm, int ts, int wtm, int tt,
                                                  int gstep) {
  SlotLayout L;
  L.xs = 0;
  L.ws = xs ? ((ftm + gstep) * fsp + 3) / 4 * 4 : 0;
  L.gs = L.ws + (wsm + 3) / 4 * 4;
  L.wt = L.gs + 2 * ts;
  L.gt = L.wt + (wtm + 3) / 4 * 4;
  L.per = L.gt + 2 * tt;
  return L;
}

struct TermHdr {
  long long src_off;
  float scale;
  int fs_lo, fs_w, ws_off, ft_lo, ft_w, wt_off, s_tab, t_tab;
};

// 16 FFMAs: acc[r][c] += w[r] * u[c]
__device__ __forceinline__ void fma4x4(float (&acc)[4][4], const float4 w4, const float4 u4) {
  acc[0][0] = fmaf(w4.x, u4.x, acc[0][0]); acc[0][1] = fmaf(w4.x, u4.y, acc[0][1]);
  acc[0][2] = fmaf(w4.x, u4.z, acc[0][2]); acc[0][3] = fmaf(w4.x, u4.w, acc[0][3]);
  acc[1][0] = fmaf(w4.y, u4.x, acc[1][0]); acc[1][1] = fmaf(w4.y, u4.y, acc[1][1]);
  acc[1][2] = fmaf(w4.y, u4.z, acc[1][2]); acc[1][3] = fmaf(w4.y, u4.w, acc[1][3]);
  acc[2][0] = fmaf(w4.z, u4.x, acc[2][0]); acc[2][1] = fmaf(w4.z, u4.y, acc[2][1]);
  acc[2][2] = fmaf(w4.z, u4.z, acc[2][2]); acc[2][3] = fmaf(w4.z, u4.w, acc[2][3]);
  acc[3][0] = fmaf(w4.w, u4.x, acc[3][0]); acc[3][1] = fmaf(w4.w, u4.y, acc[3][1]);
  acc[3][2] = fmaf(w4.w, u4.z, acc[3][2]); acc[3][3] = fmaf(w4.w, u4.w, acc[3][3]);
}

// MODE 0: source footprint staged in smem, pass 1 from smem;  MODE 1: pass 1 gathers from L1/L2;
// MODE 2: identity s table, source rows staged straight into U;  MODE 3: identity s table, pass 2
// streams the source rows from L1/L2 (no U tile).
template <int TS, int TT, int NT, int MODE>
__global__ void __launch_bounds__(NT, 640 / NT) sep_kernel(SepArgs a) {
  constexpr int NQ = TS / 4;           // 4-column groups per tile (pass 1 groups, pass 2 quads)
  constexpr int GSTEP = NT / NQ;       // pass 2: row groups in flight; pass 1: row stride
  constexpr int NG = TT / 4;           // row groups per tile
  constexpr int GP = NG / GSTEP;       // row groups per thread in pass 2
  constexpr bool XS = MODE == 0;
  constexpr bool IDENT = MODE >= 2;
  static_assert(GP >= 1 && NG % GSTEP == 0 && NT % NQ == 0, "tile/thread mismatch");
  extern __shared__ __align__(16) float smem[];
  __shared__ TermHdr hdr[2][8];
  const int tid = threadIdx.x;
  const int tx = blockIdx.x, ty = blockIdx.y + a.ty0, b = blockIdx.z;
  const int os0 = tx * TS, ot0 = ty * TT;
  const SlotLayout L = slot_layout(a.ftm, a.fsp, XS, a.wsm, TS, a.wtm, TT, GSTEP);
  const int urows = a.ftm + GSTEP;  // U tile rows (padded)
  const int nbuf = a.nbuf;
  float* bufs[2] = {smem, smem + (nbuf - 1) * a.nb * L.per};
  float* Ubase = smem + nbuf * a.nb * L.per;   // [nbuf][nb][urows][TS]
  const int quad = tid % NQ, gsub = tid / NQ;

  float acc[GP][4][4];
#pragma unroll
  for (int j = 0; j < GP; ++j)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[j][r][c] = 0.f;

  const int e0 = a.offs[b], e1 = a.offs[b + 1];
  const int nchunks = (e1 - e0 + a.nb - 1) / a.nb;

  auto stage_chunk = [&](int ci, int sd) {
    const int e = e0 + ci * a.nb;
    const int nterm = min(a.nb, e1 - e);
    float* buf = bufs[sd];
    for (int sl = 0; sl < nterm; ++sl) {
      const Term term = a.terms[e + sl];
      const TileT fs = a.fp_s[(size_t)term.s_tab * a.ntx + tx];
      const TileT ft = a.fp_t[(size_t)term.t_tab * a.nty + ty];
      const bool live = fs.width != 0 && ft.width != 0 && ft.lo < a.win_r1 && ft.lo + ft.width > a.win_r0;
      const bool windowed = ft.lo < a.win_r0 || ft.lo + ft.width > a.win_r1;
      if (tid == 0) {
        TermHdr h;
        h.src_off = term.src_off;
        h.scale = term.scale;
        h.fs_lo = fs.lo;
        h.fs_w = live ? fs.width : 0;
        h.ws_off = fs.woff;
        h.ft_lo = ft.lo;
        h.ft_w = ft.width;
        h.wt_off = ft.woff;
        h.s_tab = term.s_tab;
        h.t_tab = term.t_tab;
        hdr[sd][sl] = h;
      }
      if (!live) continue;
      float* slot = buf + sl * L.per;
      if (MODE == 2) {
        // U[r][c] = src[ft.lo + r][os0 + c]
        float* U = Ubase + (size_t)((sd % nbuf) * a.nb + sl) * urows * TS;
        const float* src = a.src + term.src_off + os0;
        const int ncol = min(TS, a.n_is - os0);
        if (((a.n_is & 3) == 0) && ((a.src_pitch & 3) == 0) && ((term.src_off & 3) == 0) && ncol == TS && !windowed) {
          for (int q = tid; q < ft.width * NQ; q += NT) {
            const int r = q / NQ, c4 = q - r * NQ;
            __pipeline_memcpy_async(U + r * TS + 4 * c4, src + (size_t)(ft.lo + r) * a.src_pitch + 4 * c4, 16);
          }
        } else {
          for (int q = tid; q < ft.width * TS; q += NT) {
            const int r = q / TS, c = q - r * TS;
            const int row = ft.lo + r;
            if (c < ncol && row >= a.win_r0 && row < a.win_r1)
              __pipeline_memcpy_async(U + r * TS + c, src + (size_t)row * a.src_pitch + c, 4);
            else
              U[r * TS + c] = 0.f;
          }
        }
      }
      if (XS) {
        const float* src = a.src + term.src_off + fs.lo;
        const int n = ft.width * fs.width;
        for (int q = tid; q < n; q += NT) {
          const int r = q / fs.width, c = q - r * fs.width;
          const int row = ft.lo + r;
          if (!windowed || (row >= a.win_r0 && row < a.win_r1))
            __pipeline_memcpy_async(slot + L.xs + r * a.fsp + c, src + (size_t)row * a.src_pitch + c, 4);
          else
            slot[L.xs + r * a.fsp + c] = 0.f;
        }
      }
      if (!IDENT) {
        for (int q = tid; q < fs.wlen / 4; q += NT)
          __pipeline_memcpy_async(slot + L.ws + 4 * q, a.s_gw + fs.woff + 4 * q, 16);
        const int g0 = tx * NQ;
        for (int q = tid; q < 2 * NQ; q += NT) {
          if (g0 + q / 2 < a.s_ngroups)
            __pipeline_memcpy_async(slot + L.gs + 4 * q, a.s_g + 2 * ((size_t)term.s_tab * a.s_ngroups + g0) + q, 16);
          else
            reinterpret_cast<int4*>(slot + L.gs)[q] = make_int4(0, 0, 0, 0);
        }
      }
      for (int q = tid; q < ft.wlen / 4; q += NT)
        __pipeline_memcpy_async(slot + L.wt + 4 * q, a.t_gw + ft.woff + 4 * q, 16);
      const int g0 = ty * NG;
      for (int q = tid; q < 2 * NG; q += NT) {
        if (g0 + q / 2 < a.t_ngroups)
          __pipeline_memcpy_async(slot + L.gt + 4 * q, a.t_g + 2 * ((size_t)term.t_tab * a.t_ngroups + g0) + q, 16);
        else
          reinterpret_cast<int4*>(slot + L.gt)[q] = make_int4(0, 0, 0, 0);
      }
    }
    __pipeline_commit();
  };

  if (nchunks > 0) stage_chunk(0, 0);
  for (int ci = 0; ci < nchunks; ++ci) {
    const int sd = ci & 1;
    const int nterm = min(a.nb, e1 - (e0 + ci * a.nb));
    float* buf = bufs[sd];
    if (ci + 1 < nchunks) {
      stage_chunk(ci + 1, sd ^ 1);
      __pipeline_wait_prior(1);
    } else {
      __pipeline_wait_prior(0);
    }
    __syncthreads();
    // ---- pass 1 (s direction, G4 segments): thread = (column group `quad`, rows gsub, gsub+GSTEP, ...)
    if (!IDENT) {
      for (int sl = 0; sl < nterm; ++sl) {
        const TermHdr h = hdr[sd][sl];
        if (h.fs_w == 0) continue;
        const float* slot = buf + sl * L.per;
        float* U = Ubase + (size_t)((sd % nbuf) * a.nb + sl) * urows * TS;
        const int4* GS = reinterpret_cast<const int4*>(slot + L.gs);
        const int4 sg0 = GS[2 * quad], sg1 = GS[2 * quad + 1];
        const long long pitch = XS ? a.fsp : a.src_pitch;
        const float* xbase = XS ? slot + L.xs - h.fs_lo : a.src + h.src_off + (size_t)h.ft_lo * a.src_pitch;
        // two rows per step; staged rows are padded so the second row is always addressable
        for (int r0 = gsub; r0 < h.ft_w; r0 += 2 * GSTEP) {
          float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
          const bool in0 = XS || (h.ft_lo + r0 >= a.win_r0 && h.ft_lo + r0 < a.win_r1);
          const bool two = r0 + GSTEP < h.ft_w;
          const bool in1 = XS || (two && h.ft_lo + r0 + GSTEP >= a.win_r0 && h.ft_lo + r0 + GSTEP < a.win_r1);
#pragma unroll
          for (int sgi = 0; sgi < 2; ++sgi) {
            const int4 sg = sgi ? sg1 : sg0;
            const float4* wp = reinterpret_cast<const float4*>(slot + L.ws + (sg.z - h.ws_off));
            const float* x0 = xbase + (size_t)r0 * pitch + sg.x;
            const float* x1 = x0 + (size_t)GSTEP * pitch;
#pragma unroll 4
            for (int p = 0; p < sg.y; ++p) {
              const float4 w4 = wp[p];
              const float a0 = XS ? x0[p] : (in0 ? __ldg(x0 + p) : 0.f);
              const float a1 = XS ? x1[p] : (in1 ? __ldg(x1 + p) : 0.f);
              v0.x = fmaf(w4.x, a0, v0.x); v0.y = fmaf(w4.y, a0, v0.y);
              v0.z = fmaf(w4.z, a0, v0.z); v0.w = fmaf(w4.w, a0, v0.w);
              v1.x = fmaf(w4.x, a1, v1.x); v1.y = fmaf(w4.y, a1, v1.y);
              v1.z = fmaf(w4.z, a1, v1.z); v1.w = fmaf(w4.w, a1, v1.w);
            }
          }
          v0.x *= h.scale; v0.y *= h.scale; v0.z *= h.scale; v0.w *= h.scale;
          v1.x *= h.scale; v1.y *= h.scale; v1.z *= h.scale; v1.w *= h.scale;
          *reinterpret_cast<float4*>(U + r0 * TS + 4 * quad) = v0;
          if (XS || two) *reinterpret_cast<float4*>(U + (r0 + GSTEP) * TS + 4 * quad) = v1;
        }
      }
    }
    if (MODE != 3) __syncthreads();
    // ---- pass 2 (t direction, G4 segments): groups of 4 output rows x 4 columns per thread
    for (int sl = 0; sl < nterm; ++sl) {
      const TermHdr h = hdr[sd][sl];
      if (h.fs_w == 0) continue;
      const float* slot = buf + sl * L.per;
      const int4* GD = reinterpret_cast<const int4*>(slot + L.gt);
#pragma unroll
      for (int j = 0; j < GP; ++j) {
        const int gl = gsub + j * GSTEP;
#pragma unroll
        for (int sgi = 0; sgi < 2; ++sgi) {
          const int4 gd = GD[2 * gl + sgi];
          const float4* wp = reinterpret_cast<const float4*>(slot + L.wt + (gd.z - h.wt_off));
          if (MODE != 3) {
            const float* U = Ubase + (size_t)((sd % nbuf) * a.nb + sl) * urows * TS;
            const float4* up = reinterpret_cast<const float4*>(U + (gd.x - h.ft_lo) * TS + quad * 4);
#pragma unroll 4
            for (int p = 0; p < gd.y; ++p) fma4x4(acc[j], wp[p], up[p * (TS / 4)]);
          } else {
            const int gcol = os0 + quad * 4;
            const bool gvec = ((a.n_is & 3) == 0) && ((a.src_pitch & 3) == 0) && ((h.src_off & 3) == 0) && gcol + 3 < a.n_is;
            const float* gp = a.src + h.src_off + (size_t)gd.x * a.src_pitch + gcol;
#pragma unroll 4
            for (int p = 0; p < gd.y; ++p) {
              const int row = gd.x + p;
              const bool rin = row >= a.win_r0 && row < a.win_r1;
              float4 u4 = make_float4(0.f, 0.f, 0.f, 0.f);
              if (rin) {
                if (gvec) {
                  u4 = __ldg(reinterpret_cast<const float4*>(gp + (size_t)p * a.src_pitch));
                } else {
                  const float* q = gp + (size_t)p * a.src_pitch;
                  if (gcol + 0 < a.n_is) u4.x = __ldg(q + 0);
                  if (gcol + 1 < a.n_is) u4.y = __ldg(q + 1);
                  if (gcol + 2 < a.n_is) u4.z = __ldg(q + 2);
                  if (gcol + 3 < a.n_is) u4.w = __ldg(q + 3);
                }
              }
              fma4x4(acc[j], wp[p], u4);
            }
          }
        }
      }
    }
    __syncthreads();  // chunk done with U and its buffer before they are refilled
  }
  float* outb = a.out + (size_t)b * a.out_stride;
  const int col = os0 + quad * 4;
  const bool vec = (col + 3 < a.n_os) && ((a.n_os & 3) == 0) && ((a.out_pitch & 3) == 0) && ((a.out_stride & 3) == 0);
#pragma unroll
  for (int j = 0; j < GP; ++j) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = ot0 + 4 * (gsub + j * GSTEP) + r;
      if (row >= a.n_ot) continue;
      float* p = outb + (size_t)row * a.out_pitch + col;
      float v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = a.out_scale * acc[j][r][c];
      if (vec) {
        float4 o = make_float4(v[0], v[1], v[2], v[3]);
        if (a.accumulate) {
          const float4 q = *reinterpret_cast<float4*>(p);
          o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
        }
        *reinterpret_cast<float4*>(p) = o;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (col + c >= a.n_os) continue;
          p[c] = a.accumulate ? p[c] + v[c] : v[c];
        }
      }
    }
  }
}

template <int TS, int TT, int NT, int MODE>
static lfm_status launch_sep_t(const SepArgs& a, dim3 grid, size_t smem, cudaStream_t s, std::string& err) {
  auto kern = sep_kernel<TS, TT, NT, MODE>;
  static bool configured_dev[LFM_MAX_DEV];  // per instantiation and device
  bool& configured = configured_dev[cur_dev()];
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(sep_kernel)", err);
    configured = true;
  }
  kern<<<grid, NT, smem, s>>>(a);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "sep_kernel launch", err);
}

// ------------------------------------------------------------------------------------------
// Streaming t-pass for ops whose s table is the identity (collapsed forward pass 2, adjoint pass 1):
//   out[4g+q][c] (+)= scale * sum_terms sum_seg sum_p Wt_g[p][q] * src_e[j0 + p][os0 + c]
// A producer warp streams, per term, the tile's source window rows (one cp.async.bulk per row),
// the tile's weight block and group descriptors into a STAGES-deep ring of shared-memory slots,
// completing on an mbarrier (expect_tx); NCW consumer warps wait on the slot's mbarrier, run the
// 16-FFMA micro-kernel and release the slot on an "empty" mbarrier.  No CTA-wide barriers in the loop.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// L2-gather t-pass over the MSEG form of the t family (identity s): per group a CSR list of dense
// segments (one per cluster of source rows), so the FMA slots follow the non-zeros (~95% for the
// slice-interleaved adjoint family, vs ~36-52% with two segments).  L2 gather, no shared memory.
template <int GR>
__device__ __forceinline__ void fma_gr(float (&acc)[GR][4], const float* __restrict__ w, float4 u) {
#pragma unroll
  for (int q4 = 0; q4 < GR / 4; ++q4) {
    const float4 w4 = __ldg(reinterpret_cast<const float4*>(w) + q4);
    const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      acc[4 * q4 + r][0] = fmaf(wv[r], u.x, acc[4 * q4 + r][0]);
      acc[4 * q4 + r][1] = fmaf(wv[r], u.y, acc[4 * q4 + r][1]);
      acc[4 * q4 + r][2] = fmaf(wv[r], u.z, acc[4 * q4 + r][2]);
      acc[4 * q4 + r][3] = fmaf(wv[r], u.w, acc[4 * q4 + r][3]);
    }
  }
}

// GR = rows per MSEG group (4 or 8): each source load feeds GR x 4 FMAs.
template <int TS, int TT, int NT, int UNR, bool TOUT, int GR>
__global__ void __launch_bounds__(NT, (GR == 8 ? 512 : 1024) / NT) band_m_kernel(SepArgs a) {
  constexpr int NQ = TS / 4;
  constexpr int GSTEP = NT / NQ;
  constexpr int NG = TT / GR;
  constexpr int GP = NG / GSTEP;
  static_assert(GP >= 1 && NG % GSTEP == 0 && NT % NQ == 0, "tile/thread mismatch");
  const int tid = threadIdx.x;
  const int quad = tid % NQ, gsub = tid / NQ;
  const int tx = blockIdx.x, ty = blockIdx.y + a.ty0, b = blockIdx.z;
  const int os0 = tx * TS, ot0 = ty * TT;
  const int col = os0 + quad * 4;
  if (col >= a.n_is) return;  // n_is % 4 == 0 (checked at tuning time): whole quads in or out
  const int e0 = a.offs[b], e1 = a.offs[b + 1];
  const int ngroups = (a.n_ot + GR - 1) / GR;
  float acc[GP][GR][4];
#pragma unroll
  for (int j = 0; j < GP; ++j)
#pragma unroll
    for (int r = 0; r < GR; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[j][r][c] = 0.f;
  for (int e = e0; e < e1; ++e) {
    const Term term = a.terms[e];
    const float* src = a.src + term.src_off + col;
#pragma unroll
    for (int j = 0; j < GP; ++j) {
      const int g = ty * NG + gsub + j * GSTEP;
      if (g >= ngroups) continue;
      const size_t gi = (size_t)term.t_tab * ngroups + g;
      const int s0 = __ldg(a.t_moff + gi), s1 = __ldg(a.t_moff + gi + 1);
      for (int sg = s0; sg < s1; ++sg) {
        const int4 gd = __ldg(a.t_mseg + sg);
        const int p0 = max(0, a.win_r0 - gd.x), p1 = min(gd.y, a.win_r1 - gd.x);
        const float* wp = a.t_mw + gd.z;
        const float* up = src + (size_t)gd.x * a.src_pitch;
#pragma unroll UNR
        for (int p = p0; p < p1; ++p)
          fma_gr<GR>(acc[j], wp + GR * p, __ldg(reinterpret_cast<const float4*>(up + (size_t)p * a.src_pitch)));
      }
    }
  }
  float* outb = a.out + (size_t)b * a.out_stride;
  if (TOUT) {
    // transposed output: element (row, col) at outb[col * out_pitch + row]; 4 consecutive rows per store
#pragma unroll
    for (int j = 0; j < GP; ++j) {
#pragma unroll
      for (int r4 = 0; r4 < GR / 4; ++r4) {
        const int row0 = ot0 + GR * (gsub + j * GSTEP) + 4 * r4;
        if (row0 >= a.n_ot) continue;
        const bool vec =
            row0 + 3 < a.n_ot && ((a.n_ot & 3) == 0) && ((a.out_pitch & 3) == 0) && ((a.out_stride & 3) == 0);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (col + c >= a.n_os) continue;
          float* p = outb + (size_t)(col + c) * a.out_pitch + row0;
          float v[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) v[r] = a.out_scale * acc[j][4 * r4 + r][c];
          if (vec) {
            float4 o = make_float4(v[0], v[1], v[2], v[3]);
            if (a.accumulate) {
              const float4 q = *reinterpret_cast<float4*>(p);
              o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
            }
            *reinterpret_cast<float4*>(p) = o;
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              if (row0 + r >= a.n_ot) continue;
              p[r] = a.accumulate ? p[r] + v[r] : v[r];
            }
          }
        }
      }
    }
    return;
  }
  const bool vec = (col + 3 < a.n_os) && ((a.n_os & 3) == 0) && ((a.out_pitch & 3) == 0) && ((a.out_stride & 3) == 0);
#pragma unroll
  for (int j = 0; j < GP; ++j) {
#pragma unroll
    for (int r = 0; r < GR; ++r) {
      const int row = ot0 + GR * (gsub + j * GSTEP) + r;
      if (row >= a.n_ot) continue;
      float* p = outb + (size_t)row * a.out_pitch + col;
      float v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = a.out_scale * acc[j][r][c];
      if (vec) {
        float4 o = make_float4(v[0], v[1], v[2], v[3]);
        if (a.accumulate) {
          const float4 q = *reinterpret_cast<float4*>(p);
          o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
        }
        *reinterpret_cast<float4*>(p) = o;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (col + c >= a.n_os) continue;
          p[c] = a.accumulate ? p[c] + v[c] : v[c];
        }
      }
    }
  }
}

// Flat L2-gather t-pass (identity s): per group of 4 output rows a padded list of entries
// (source row, 4 weights); the loop runs over blocks of 4 entries with the rows fetched as one int4,
// so 4 x (16-byte source load + 16-byte weight load) per block are independent and the unroll keeps
// UNR blocks of loads in flight.  Rows outside [win_r0, win_r1) contribute zero (predicated loads).
template <int TS, int TT, int NT, int UNR, bool TOUT>
__global__ void __launch_bounds__(NT, 1024 / NT) band_f_kernel(SepArgs a) {
  constexpr int NQ = TS / 4;
  constexpr int GSTEP = NT / NQ;
  constexpr int NG = TT / 4;
  constexpr int GP = NG / GSTEP;
  static_assert(GP >= 1 && NG % GSTEP == 0 && NT % NQ == 0, "tile/thread mismatch");
  const int tid = threadIdx.x;
  const int quad = tid % NQ, gsub = tid / NQ;
  const int tx = blockIdx.x, ty = blockIdx.y + a.ty0, b = blockIdx.z;
  const int os0 = tx * TS, ot0 = ty * TT;
  const int col = os0 + quad * 4;
  if (col >= a.n_is) return;
  const int e0 = a.offs[b], e1 = a.offs[b + 1];
  const bool windowed = a.win_r0 > 0 || a.win_r1 < a.n_it;
  float acc[GP][4][4];
#pragma unroll
  for (int j = 0; j < GP; ++j)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[j][r][c] = 0.f;
  for (int e = e0; e < e1; ++e) {
    const Term term = a.terms[e];
    const float* src = a.src + term.src_off + col;
#pragma unroll
    for (int j = 0; j < GP; ++j) {
      const int g = ty * NG + gsub + j * GSTEP;
      if (g >= a.t_ngroups) continue;
      const size_t gi = (size_t)term.t_tab * a.t_ngroups + g;
      const int q0 = __ldg(a.t_foff + gi) / 4, q1 = __ldg(a.t_foff + gi + 1) / 4;
      if (!windowed) {
#pragma unroll UNR
        for (int q = q0; q < q1; ++q) {
          const int4 rw = __ldg(a.t_frow + q);
          const float4 u0 = __ldg(reinterpret_cast<const float4*>(src + (size_t)rw.x * a.src_pitch));
          const float4 u1 = __ldg(reinterpret_cast<const float4*>(src + (size_t)rw.y * a.src_pitch));
          const float4 u2 = __ldg(reinterpret_cast<const float4*>(src + (size_t)rw.z * a.src_pitch));
          const float4 u3 = __ldg(reinterpret_cast<const float4*>(src + (size_t)rw.w * a.src_pitch));
          fma4x4(acc[j], __ldg(a.t_fw + 4 * q + 0), u0);
          fma4x4(acc[j], __ldg(a.t_fw + 4 * q + 1), u1);
          fma4x4(acc[j], __ldg(a.t_fw + 4 * q + 2), u2);
          fma4x4(acc[j], __ldg(a.t_fw + 4 * q + 3), u3);
        }
      } else {
        // row window (adjoint detector-row sharding): entries are in increasing row order within the group,
        // so only the blocks of 4 entries that straddle or lie inside [win_r0, win_r1) are visited
        const int* fr = reinterpret_cast<const int*>(a.t_frow);
        int lo = q0, hi = q1;  // first block whose last row >= win_r0, first block whose first row >= win_r1
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (__ldg(fr + 4 * mid + 3) < a.win_r0) lo = mid + 1; else hi = mid;
        }
        int lo2 = lo, hi2 = q1;
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (__ldg(fr + 4 * mid) < a.win_r1) lo2 = mid + 1; else hi2 = mid;
        }
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll UNR
        for (int q = lo; q < lo2; ++q) {
          const int4 rw = __ldg(a.t_frow + q);
          const bool i0 = rw.x >= a.win_r0 && rw.x < a.win_r1, i1 = rw.y >= a.win_r0 && rw.y < a.win_r1;
          const bool i2 = rw.z >= a.win_r0 && rw.z < a.win_r1, i3 = rw.w >= a.win_r0 && rw.w < a.win_r1;
          const float4 u0 = i0 ? __ldg(reinterpret_cast<const float4*>(src + (size_t)rw.x * a.src_pitch)) : z;
          const float4 u1 = i1 ? __ldg(reinterpret_cast<const float4*>(src + (size_t)rw.y * a.src_pitch)) : z;
          const float4 u2 = i2 ? __ldg(reinterpret_cast<const float4*>(src + (size_t)rw.z * a.src_pitch)) : z;
          const float4 u3 = i3 ? __ldg(reinterpret_cast<const float4*>(src + (size_t)rw.w * a.src_pitch)) : z;
          fma4x4(acc[j], __ldg(a.t_fw + 4 * q + 0), u0);
          fma4x4(acc[j], __ldg(a.t_fw + 4 * q + 1), u1);
          fma4x4(acc[j], __ldg(a.t_fw + 4 * q + 2), u2);
          fma4x4(acc[j], __ldg(a.t_fw + 4 * q + 3), u3);
        }
      }
    }
  }
  float* outb = a.out + (size_t)b * a.out_stride;
  if (TOUT) {
#pragma unroll
    for (int j = 0; j < GP; ++j) {
      const int row0 = ot0 + 4 * (gsub + j * GSTEP);
      if (row0 >= a.n_ot) continue;
      const bool vec = row0 + 3 < a.n_ot && ((a.n_ot & 3) == 0) && ((a.out_pitch & 3) == 0) && ((a.out_stride & 3) == 0);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (col + c >= a.n_os) continue;
        float* p = outb + (size_t)(col + c) * a.out_pitch + row0;
        float v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) v[r] = a.out_scale * acc[j][r][c];
        if (vec) {
          float4 o = make_float4(v[0], v[1], v[2], v[3]);
          if (a.accumulate) {
            const float4 q = *reinterpret_cast<float4*>(p);
            o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
          }
          *reinterpret_cast<float4*>(p) = o;
        } else {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (row0 + r >= a.n_ot) continue;
            p[r] = a.accumulate ? p[r] + v[r] : v[r];
          }
        }
      }
    }
    return;
  }
  const bool vec = (col + 3 < a.n_os) && ((a.n_os & 3) == 0) && ((a.out_pitch & 3) == 0) && ((a.out_stride & 3) == 0);
#pragma unroll
  for (int j = 0; j < GP; ++j) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = ot0 + 4 * (gsub + j * GSTEP) + r;
      if (row >= a.n_ot) continue;
      float* p = outb + (size_t)row * a.out_pitch + col;
      float v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = a.out_scale * acc[j][r][c];
      if (vec) {
        float4 o = make_float4(v[0], v[1], v[2], v[3]);
        if (a.accumulate) {
          const float4 q = *reinterpret_cast<float4*>(p);
          o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
        }
        *reinterpret_cast<float4*>(p) = o;
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (col + c >= a.n_os) continue;
          p[c] = a.accumulate ? p[c] + v[c] : v[c];
        }
      }
    }
  }
}

template <int TS, int TT, int NT>
static lfm_status launch_band_f(const SepArgs& a, dim3 grid, cudaStream_t s, std::string& err, int unr, int tout) {
  if (tout) {
    if (unr == 2)
      band_f_kernel<TS, TT, NT, 2, true><<<grid, NT, 0, s>>>(a);
    else
      band_f_kernel<TS, TT, NT, 1, true><<<grid, NT, 0, s>>>(a);
  } else if (unr == 2) {
    band_f_kernel<TS, TT, NT, 2, false><<<grid, NT, 0, s>>>(a);
  } else {
    band_f_kernel<TS, TT, NT, 1, false><<<grid, NT, 0, s>>>(a);
  }
  ++g_launches;
  return cuda_check(cudaGetLastError(), "band_f_kernel launch", err);
}

template <int TS, int TT, int NT>
static lfm_status launch_band_m8(const SepArgs& a, dim3 grid, cudaStream_t s, std::string& err, int unr, int tout) {
  if (tout) {
    if (unr == 8)
      band_m_kernel<TS, TT, NT, 8, true, 8><<<grid, NT, 0, s>>>(a);
    else
      band_m_kernel<TS, TT, NT, 4, true, 8><<<grid, NT, 0, s>>>(a);
  } else if (unr == 8) {
    band_m_kernel<TS, TT, NT, 8, false, 8><<<grid, NT, 0, s>>>(a);
  } else {
    band_m_kernel<TS, TT, NT, 4, false, 8><<<grid, NT, 0, s>>>(a);
  }
  ++g_launches;
  return cuda_check(cudaGetLastError(), "band_m_kernel launch", err);
}

template <int TS, int TT, int NT>
static lfm_status launch_band_m(const SepArgs& a, dim3 grid, cudaStream_t s, std::string& err, int unr, int tout) {
  if (tout) {
    if (unr == 8)
      band_m_kernel<TS, TT, NT, 8, true, 4><<<grid, NT, 0, s>>>(a);
    else
      band_m_kernel<TS, TT, NT, 4, true, 4><<<grid, NT, 0, s>>>(a);
  } else if (unr == 8) {
    band_m_kernel<TS, TT, NT, 8, false, 4><<<grid, NT, 0, s>>>(a);
  } else {
    band_m_kernel<TS, TT, NT, 4, false, 4><<<grid, NT, 0, s>>>(a);
  }
  ++g_launches;
  return cuda_check(cudaGetLastError(), "band_m_kernel launch", err);
}

__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ in, float* __restrict__ out, int R,
                                                        int C, long long in_bs, long long in_pitch, long long out_bs,
                                                        long long out_pitch) {
  __shared__ float tile[32][33];
  const int b = blockIdx.z;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const float* ib = in + (size_t)b * in_bs;
  float* ob = out + (size_t)b * out_bs;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int r = r0 + ty + k, c = c0 + tx;
    if (r < R && c < C) tile[ty + k][tx] = ib[(size_t)r * in_pitch + c];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int c = c0 + ty + k, r = r0 + tx;
    if (r < R && c < C) ob[(size_t)c * out_pitch + r] = tile[tx][ty + k];
  }
}

// 64 x 64 tiles with 16-byte accesses on both sides (rows and pitches multiples of 4 floats, 16-byte aligned
// bases): 4 KB in flight per warp instead of 512 B.
__global__ void __launch_bounds__(256) transpose64_kernel(const float* __restrict__ in, float* __restrict__ out, int R,
                                                          int C, long long in_bs, long long in_pitch, long long out_bs,
                                                          long long out_pitch) {
  __shared__ float tile[64][65];
  const int b = blockIdx.z;
  const int c0 = blockIdx.x * 64, r0 = blockIdx.y * 64;
  const float* ib = in + (size_t)b * in_bs;
  float* ob = out + (size_t)b * out_bs;
  const int t = threadIdx.x;
  const int lc = 4 * (t & 15), lr = t >> 4;
  float4 v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = r0 + lr + 16 * k, c = c0 + lc;
    v[k] = (r < R && c < C) ? __ldg(reinterpret_cast<const float4*>(ib + (size_t)r * in_pitch + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float* d = &tile[lr + 16 * k][lc];
    d[0] = v[k].x; d[1] = v[k].y; d[2] = v[k].z; d[3] = v[k].w;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = c0 + lr + 16 * k, r = r0 + lc;
    if (r < R && c < C) {
      const float4 o = make_float4(tile[lc][lr + 16 * k], tile[lc + 1][lr + 16 * k], tile[lc + 2][lr + 16 * k],
                                   tile[lc + 3][lr + 16 * k]);
      *reinterpret_cast<float4*>(ob + (size_t)c * out_pitch + r) = o;
    }
  }
}

lfm_status k_transpose(const float* in, float* out, int B, int R, int C, long long in_bs, long long in_pitch,
                       long long out_bs, long long out_pitch, void* stream, std::string& err) {
  if (B <= 0 || R <= 0 || C <= 0) return LFM_OK;
  if (R % 4 == 0 && C % 4 == 0 && in_bs % 4 == 0 && in_pitch % 4 == 0 && out_bs % 4 == 0 && out_pitch % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(in) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    dim3 g64((C + 63) / 64, (R + 63) / 64, B);
    transpose64_kernel<<<g64, 256, 0, (cudaStream_t)stream>>>(in, out, R, C, in_bs, in_pitch, out_bs, out_pitch);
    ++g_launches;
    return cuda_check(cudaGetLastError(), "transpose64_kernel launch", err);
  }
  dim3 grid((C + 31) / 32, (R + 31) / 32, B);
  transpose_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(in, out, R, C, in_bs, in_pitch, out_bs, out_pitch);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "transpose_kernel launch", err);
}

// Quarter-turn relabelling (reading R7): out[I] (+)= in[src(I)] with src_b = I_{axis[b]} or
// n_b - 1 - I_{axis[b]} (sign[b] < 0); exact, pure data movement (8 bytes per voxel).
struct PermMap {
  int axis[3], sign[3];
};

__global__ void permute_kernel(const float* __restrict__ in, float* __restrict__ out, int nx, int ny, int nz, PermMap m,
                               int accumulate) {
  const long long n = (long long)nx * ny * nz;
  const int dims[3] = {nx, ny, nz};
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
    const int I[3] = {(int)(v % nx), (int)((v / nx) % ny), (int)(v / ((long long)nx * ny))};
    int S[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int i = I[m.axis[b]];
      S[b] = m.sign[b] > 0 ? i : dims[b] - 1 - i;
    }
    const float val = __ldg(in + S[0] + (long long)nx * (S[1] + (long long)ny * S[2]));
    out[v] = accumulate ? out[v] + val : val;
  }
}

lfm_status k_permute(const float* in, float* out, int nx, int ny, int nz, const int* axis, const int* sign,
                     int accumulate, void* stream, std::string& err) {
  PermMap m;
  for (int b = 0; b < 3; ++b) { m.axis[b] = axis[b]; m.sign[b] = sign[b]; }
  const long long n = (long long)nx * ny * nz;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  permute_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(in, out, nx, ny, nz, m, accumulate);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "permute_kernel launch", err);
}

// ---------------------------------------------------------------------------------------------- band_u host side
// TMA descriptor of a row-major fp32 matrix (rows x cols, pitch in floats).  band_u reads its source in
// 32-column x 16-row boxes with the 128-byte / 32-byte-atom swizzle that the tcgen05 MN-major operand (layout
// type 1) expects (rows and columns outside the map read as zero: the row window of a sharded adjoint), and
// writes its output in 32 x 32 boxes with the 128-byte swizzle (writes outside the map are clipped).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static lfm_status encode_map_raw(CUtensorMap* map, const void* base, int cols, int rows, long long pitch, int box_c,
                                 int box_r, CUtensorMapSwizzle swz, std::string& err, bool f16);
// (pitch in elements; f16: 2-byte elements)
static lfm_status encode_map(CUtensorMap* map, const void* base, int cols, int rows, long long pitch, int box_c,
                             int box_r, CUtensorMapSwizzle swz, std::string& err, bool f16) {
  const TmapKey k = {base, {2, cols, rows, pitch, box_c, box_r, (long long)swz, f16, 0, 0, 0}};
  if (tmap_lookup(k, map)) return LFM_OK;
  lfm_status st = encode_map_raw(map, base, cols, rows, pitch, box_c, box_r, swz, err, f16);
  if (st == LFM_OK) tmap_insert(k, *map);
  return st;
}
static lfm_status encode_map_raw(CUtensorMap* map, const void* base, int cols, int rows, long long pitch, int box_c,
                                 int box_r, CUtensorMapSwizzle swz, std::string& err, bool f16) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &qr) != cudaSuccess ||
        !encode) {
      cudaGetLastError();
      err = "band_u: cuTensorMapEncodeTiled unavailable";
      return LFM_E_CUDA;
    }
  }
  const int esz = f16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((pitch * esz) & 15)) {
    err = "band_u: buffers and their rows must be 16-byte aligned";
    return LFM_E_INVALID;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstr[1] = {(cuuint64_t)pitch * esz};
  cuuint32_t box[2] = {(cuuint32_t)box_c, (cuuint32_t)box_r}, es[2] = {1, 1};
  CUresult r = encode(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), gdim, gstr, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "band_u: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return LFM_E_CUDA;
  }
  return LFM_OK;
}
static int g_num_sms() {
  static int sms[LFM_MAX_DEV];
  const int dev = cur_dev();
  int& n = sms[dev];
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// split-K partial sums of band_u: y[r][c] (+)= sum_kc part[kc * kc_rows + r][c] over the window, kc ascending;
// float4 per thread (window columns, pitch and the buffers on 16-byte boundaries, checked by the caller)
__global__ void sum_chunks_kernel(const float* __restrict__ part, float* __restrict__ y, long long pitch, int r0, int r1,
                                  int c0, int c1, int ksplit, int kc_rows, int accumulate) {
  const int w4 = (c1 - c0) >> 2;
  const long long n = (long long)(r1 - r0) * w4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = r0 + (int)(i / w4), c = c0 + 4 * (int)(i % w4);
    float4 v = __ldg(reinterpret_cast<const float4*>(part + (long long)r * pitch + c));
    for (int kc = 1; kc < ksplit; ++kc) {
      const float4 p = __ldg(reinterpret_cast<const float4*>(part + ((long long)kc * kc_rows + r) * pitch + c));
      v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
    }
    float4* o = reinterpret_cast<float4*>(y + (long long)r * pitch + c);
    if (accumulate) {
      const float4 q = *o;
      v.x = q.x + v.x; v.y = q.y + v.y; v.z = q.z + v.z; v.w = q.w + v.w;
    }
    *o = v;
  }
}

// per-CTA maxima of |src[0, n)| at part[blockIdx.x]; CTA 0 zero-fills the other LFM_AMAX_SLOTS (the data scale of
// the 2xFP16 band_u form: of x^r for the forward, of y for the adjoint)
__global__ void amax_kernel(const float* __restrict__ src, long long n, float* __restrict__ part) {
  uint32_t m = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const long long n4 = n >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    long long i = i0;
    for (; i + 7 * stride < n4; i += 8 * stride) {  // eight independent loads in flight
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg(s4 + i + j * stride);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        m = max(max(max(m, __float_as_uint(v[j].x) & 0x7fffffffu), max(__float_as_uint(v[j].y) & 0x7fffffffu,
                __float_as_uint(v[j].z) & 0x7fffffffu)), __float_as_uint(v[j].w) & 0x7fffffffu);
    }
    for (; i < n4; i += stride) {
      const float4 v = __ldg(s4 + i);
      m = max(max(max(m, __float_as_uint(v.x) & 0x7fffffffu), max(__float_as_uint(v.y) & 0x7fffffffu,
              __float_as_uint(v.z) & 0x7fffffffu)), __float_as_uint(v.w) & 0x7fffffffu);
    }
    for (long long i = 4 * n4 + i0; i < n; i += stride) m = max(m, __float_as_uint(__ldg(src + i)) & 0x7fffffffu);
  } else {
    for (long long i = i0; i < n; i += stride) m = max(m, __float_as_uint(__ldg(src + i)) & 0x7fffffffu);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ uint32_t red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) part[blockIdx.x] = __uint_as_float(m);
    if (blockIdx.x == 0)
      for (int i = gridDim.x + threadIdx.x; i < LFM_AMAX_SLOTS; i += 32) part[i] = 0.f;
  }
}

lfm_status k_amax(const float* src, long long n, float* part, void* stream, std::string& err) {
  // enough threads that every load of a 16 MiB source is in flight at once (8 float4 per thread)
  const int g = std::min(LFM_AMAX_SLOTS, (int)std::max<long long>(1, (n / 4 + 1023) / 1024));
  amax_kernel<<<g, 1024, 0, (cudaStream_t)stream>>>(src, n, part);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "amax_kernel launch", err);
}

// fp16 hi / lo of 2^e src (e from the partial maxima of |src|, as band_u computes it); float4 path when aligned
__global__ void split16_kernel(const float* __restrict__ src, long long n, const float* __restrict__ amax,
                               uint16_t* __restrict__ hi, uint16_t* __restrict__ lo) {
  const float sig = pow2f(u_data_exp(amax, LFM_AMAX_SLOTS, 1.f));
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo)) & 15) == 0;
  const long long n4 = vec ? n >> 2 : 0;
  auto one = [&](long long i, const float4 v) {
    const float x0 = sig * v.x, x1 = sig * v.y, x2 = sig * v.z, x3 = sig * v.w;
    const __half2 h01 = __floats2half2_rn(x0, x1), h23 = __floats2half2_rn(x2, x3);
    const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
    const __half2 l01 = __floats2half2_rn(x0 - f01.x, x1 - f01.y), l23 = __floats2half2_rn(x2 - f23.x, x3 - f23.y);
    reinterpret_cast<uint2*>(hi)[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
    reinterpret_cast<uint2*>(lo)[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
  };
  long long i = i0;
  for (; i + 3 * stride < n4; i += 4 * stride) {  // four independent loads in flight
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = __ldg(reinterpret_cast<const float4*>(src) + i + j * stride);
#pragma unroll
    for (int j = 0; j < 4; ++j) one(i + j * stride, v[j]);
  }
  for (; i < n4; i += stride) one(i, __ldg(reinterpret_cast<const float4*>(src) + i));
  for (long long i = 4 * n4 + i0; i < n; i += stride) {
    const float x = sig * __ldg(src + i);
    const __half h = __float2half_rn(x), l = __float2half_rn(x - __half2float(h));
    hi[i] = *reinterpret_cast<const uint16_t*>(&h);
    lo[i] = *reinterpret_cast<const uint16_t*>(&l);
  }
}

// Row-scaled fp16 split in one pass (the A operand of band_v's 2xFP16 forward, whose rows are the MMA's M rows, so a
// scale per row is undone per output row): one warp per row of `len` floats, e_row from the row's maximum
// (u_data_exp), hi / lo of 2^e_row src, rinv[row] = 2^-e_row; the per-CTA maxima of |src| go to part (CTA 0
// zero-fills the other LFM_AMAX_SLOTS) for the global scale of the next stage.
__global__ void split16_rows_kernel(const float* __restrict__ src, int rows, int len, float* __restrict__ part,
                                    float* __restrict__ rinv, uint16_t* __restrict__ hi, uint16_t* __restrict__ lo) {
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  const bool vec = (len & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && (len & 7) == 0;
  uint32_t cmax = 0;
  if (vec && len <= 128) {  // one float4 per lane and row: 4 rows per warp with their loads in flight together
    constexpr int RB = 4;
    const int nw = gridDim.x * wpb;
    for (int r0 = (blockIdx.x * wpb + (threadIdx.x >> 5)) * RB; r0 < rows; r0 += nw * RB) {
      float4 v[RB];
      const bool on = 4 * lane < len;
#pragma unroll
      for (int i = 0; i < RB; ++i)
        v[i] = on && r0 + i < rows ? __ldg(reinterpret_cast<const float4*>(src + (long long)(r0 + i) * len) + lane)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int row = r0 + i;
        uint32_t m = max(max(__float_as_uint(v[i].x) & 0x7fffffffu, __float_as_uint(v[i].y) & 0x7fffffffu),
                         max(__float_as_uint(v[i].z) & 0x7fffffffu, __float_as_uint(v[i].w) & 0x7fffffffu));
#pragma unroll
        for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (row >= rows) continue;  // (uniform across the warp)
        cmax = max(cmax, m);
        const int e = data_exp(__uint_as_float(m));
        const float sig = pow2f(e);
        if (lane == 0) rinv[row] = pow2f(-e);
        if (on) {
          const float x0 = sig * v[i].x, x1 = sig * v[i].y, x2 = sig * v[i].z, x3 = sig * v[i].w;
          const __half2 h01 = __floats2half2_rn(x0, x1), h23 = __floats2half2_rn(x2, x3);
          const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
          const __half2 l01 = __floats2half2_rn(x0 - f01.x, x1 - f01.y), l23 = __floats2half2_rn(x2 - f23.x, x3 - f23.y);
          const long long o4 = (long long)row * len + 4 * lane;
          *reinterpret_cast<uint2*>(hi + o4) = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
          *reinterpret_cast<uint2*>(lo + o4) = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
        }
      }
    }
  } else
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < rows; row += gridDim.x * wpb) {
    const float* r = src + (long long)row * len;
    uint32_t m = 0;
    if (vec) {
      for (int c = 4 * lane; c < len; c += 128) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(r + c));
        m = max(max(max(m, __float_as_uint(v.x) & 0x7fffffffu), max(__float_as_uint(v.y) & 0x7fffffffu,
                __float_as_uint(v.z) & 0x7fffffffu)), __float_as_uint(v.w) & 0x7fffffffu);
      }
    } else {
      for (int c = lane; c < len; c += 32) m = max(m, __float_as_uint(__ldg(r + c)) & 0x7fffffffu);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    cmax = max(cmax, m);
    const int e = data_exp(__uint_as_float(m));
    const float sig = pow2f(e);
    if (lane == 0) rinv[row] = pow2f(-e);
    uint16_t* h = hi + (long long)row * len;
    uint16_t* l = lo + (long long)row * len;
    if (vec) {
      for (int c = 4 * lane; c < len; c += 128) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(r + c));
        const float x0 = sig * v.x, x1 = sig * v.y, x2 = sig * v.z, x3 = sig * v.w;
        const __half2 h01 = __floats2half2_rn(x0, x1), h23 = __floats2half2_rn(x2, x3);
        const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
        const __half2 l01 = __floats2half2_rn(x0 - f01.x, x1 - f01.y), l23 = __floats2half2_rn(x2 - f23.x, x3 - f23.y);
        *reinterpret_cast<uint2*>(h + c) = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
        *reinterpret_cast<uint2*>(l + c) = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
      }
    } else {
      for (int c = lane; c < len; c += 32) {
        const float x = sig * __ldg(r + c);
        const __half hh = __float2half_rn(x), ll = __float2half_rn(x - __half2float(hh));
        h[c] = *reinterpret_cast<const uint16_t*>(&hh);
        l[c] = *reinterpret_cast<const uint16_t*>(&ll);
      }
    }
  }
  __shared__ uint32_t red[32];
  if (lane == 0) red[threadIdx.x >> 5] = cmax;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t m = threadIdx.x < (unsigned)wpb ? red[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) part[blockIdx.x] = __uint_as_float(m);
    if (blockIdx.x == 0)
      for (int i = gridDim.x + threadIdx.x; i < LFM_AMAX_SLOTS; i += 32) part[i] = 0.f;
  }
}

// Column-scaled fp16 split in one pass (the adjoint t pass's input y: the t pass mixes rows, never columns, so a
// scale per column is undone per output column by band_u's epilogue): a CTA owns strips of SPLITC_SC columns over
// all `rows` rows; the first SPLITC_KEEP float4 of each thread stay in registers (the whole strip for rows <=
// SPLITC_KEEP * SPLITC_RSTEP, so y is read once), e_c = data_exp(max_c), cinv[c] = 2^-e_c, then fp16 hi / lo of
// 2^e_c src.  The per-CTA maxima go to part (CTA 0 zero-fills the other LFM_AMAX_SLOTS) for the global scale of
// the t pass's fp16 output.  Needs cols % 4 == 0 and 16-byte aligned src / hi / lo rows (pitch = cols); cinv is
// padded with 1 up to cols_pad.
constexpr int SPLITC_THREADS = 512, SPLITC_SC = 16, SPLITC_QN = SPLITC_SC / 4, SPLITC_RSTEP = SPLITC_THREADS / SPLITC_QN,
              SPLITC_KEEP = 16;
__device__ __forceinline__ void split_store(uint16_t* hi, uint16_t* lo, long long o, float4 v, float4 sg) {
  const float x0 = sg.x * v.x, x1 = sg.y * v.y, x2 = sg.z * v.z, x3 = sg.w * v.w;
  const __half2 h01 = __floats2half2_rn(x0, x1), h23 = __floats2half2_rn(x2, x3);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn(x0 - f01.x, x1 - f01.y), l23 = __floats2half2_rn(x2 - f23.x, x3 - f23.y);
  *reinterpret_cast<uint2*>(hi + o) = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  *reinterpret_cast<uint2*>(lo + o) = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
}
__device__ __forceinline__ void amax4(uint32_t (&m)[4], float4 v) {
  m[0] = max(m[0], __float_as_uint(v.x) & 0x7fffffffu);
  m[1] = max(m[1], __float_as_uint(v.y) & 0x7fffffffu);
  m[2] = max(m[2], __float_as_uint(v.z) & 0x7fffffffu);
  m[3] = max(m[3], __float_as_uint(v.w) & 0x7fffffffu);
}
// RES: the source is the PWLS residual r = w (Ax - gamma_cam y), computed from its three inputs on the load (the
// arithmetic of residual_kernel), so r is never written and re-read (the residual fused into the
// adjoint's input load).
struct ResIn {
  const float* Ax = nullptr;
  const float* y = nullptr;
  const float* w = nullptr;
  const double* gamma = nullptr;
  int cam = 0;
};
template <bool RES>
__device__ __forceinline__ float4 split_src(const float* __restrict__ src, const ResIn& ri, float gm, long long o) {
  if constexpr (!RES) {
    return __ldg(reinterpret_cast<const float4*>(src + o));
  } else {
    const float4 a = __ldg(reinterpret_cast<const float4*>(ri.Ax + o));
    const float4 b = __ldg(reinterpret_cast<const float4*>(ri.y + o));
    const float4 c = __ldg(reinterpret_cast<const float4*>(ri.w + o));
    auto one = [&](float av, float bv, float cv) {
      const float d = av - gm * bv;
      return cv * d;
    };
    return make_float4(one(a.x, b.x, c.x), one(a.y, b.y, c.y), one(a.z, b.z, c.z), one(a.w, b.w, c.w));
  }
}
template <bool RES>
__global__ void __launch_bounds__(SPLITC_THREADS) split16_cols_kernel(const float* __restrict__ src, int rows, int cols,
                                                                      int cols_pad, float* __restrict__ part,
                                                                      float* __restrict__ cinv, uint16_t* __restrict__ hi,
                                                                      uint16_t* __restrict__ lo, ResIn ri) {
  const float gm = RES ? (float)ri.gamma[ri.cam] : 0.f;
  __shared__ uint32_t red[SPLITC_THREADS / 32][SPLITC_SC];
  __shared__ float csig[SPLITC_SC];
  const int t = threadIdx.x, lane = t & 31, wp = t >> 5, q = t % SPLITC_QN, r_first = t / SPLITC_QN;
  const int nstrips = (cols + SPLITC_SC - 1) / SPLITC_SC;
  uint32_t cmax = 0;
  for (int strip = blockIdx.x; strip < nstrips; strip += gridDim.x) {
    const int c = strip * SPLITC_SC + 4 * q;  // this thread's 4 columns
    const bool live = c < cols;
    uint32_t m[4] = {0, 0, 0, 0};
    float4 keep[SPLITC_KEEP];
#pragma unroll
    for (int j = 0; j < SPLITC_KEEP; ++j) {
      const int r = r_first + j * SPLITC_RSTEP;
      keep[j] = live && r < rows ? split_src<RES>(src, ri, gm, (long long)r * cols + c) : make_float4(0, 0, 0, 0);
      amax4(m, keep[j]);
    }
    for (int r = r_first + SPLITC_KEEP * SPLITC_RSTEP; r < rows; r += SPLITC_RSTEP)  // taller strips
      if (live) amax4(m, split_src<RES>(src, ri, gm, (long long)r * cols + c));
#pragma unroll
    for (int o = SPLITC_QN; o < 32; o <<= 1)  // lanes of the same column quad
#pragma unroll
      for (int i = 0; i < 4; ++i) m[i] = max(m[i], __shfl_xor_sync(0xffffffffu, m[i], o));
    if (lane < SPLITC_QN)
#pragma unroll
      for (int i = 0; i < 4; ++i) red[wp][4 * lane + i] = m[i];
    __syncthreads();
    if (t < SPLITC_SC) {  // column strip * SC + t
      uint32_t mc = 0;
      for (int w = 0; w < SPLITC_THREADS / 32; ++w) mc = max(mc, red[w][t]);
      cmax = max(cmax, mc);
      const int e = data_exp(__uint_as_float(mc));
      csig[t] = pow2f(e);
      const int col = strip * SPLITC_SC + t;
      if (col < cols_pad) cinv[col] = col < cols ? pow2f(-e) : 1.f;
    }
    __syncthreads();
    if (live) {
      const float4 sg = make_float4(csig[4 * q], csig[4 * q + 1], csig[4 * q + 2], csig[4 * q + 3]);
#pragma unroll
      for (int j = 0; j < SPLITC_KEEP; ++j) {
        const int r = r_first + j * SPLITC_RSTEP;
        if (r < rows) split_store(hi, lo, (long long)r * cols + c, keep[j], sg);
      }
      for (int r = r_first + SPLITC_KEEP * SPLITC_RSTEP; r < rows; r += SPLITC_RSTEP)
        split_store(hi, lo, (long long)r * cols + c, split_src<RES>(src, ri, gm, (long long)r * cols + c), sg);
    }
  }
  // strip padding past the last strip (cols_pad may exceed the strips' columns)
  for (int col = nstrips * SPLITC_SC + (int)(blockIdx.x * SPLITC_THREADS + t); col < cols_pad; col += gridDim.x * SPLITC_THREADS)
    cinv[col] = 1.f;
  if (t < 32) {
    uint32_t mm = t < SPLITC_SC ? cmax : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) mm = max(mm, __shfl_xor_sync(0xffffffffu, mm, o));
    if (t == 0) part[blockIdx.x] = __uint_as_float(mm);
    if (blockIdx.x == 0)
      for (int i = gridDim.x + t; i < LFM_AMAX_SLOTS; i += 32) part[i] = 0.f;
  }
}

lfm_status k_split16_cols(const float* src, int rows, int cols, int cols_pad, float* part, float* cinv, uint16_t* hi,
                          uint16_t* lo, void* stream, std::string& err) {
  if (cols % 4 || ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo)) & 15)) {
    err = "split16_cols: columns must be a multiple of 4 and rows 16-byte aligned";
    return LFM_E_INVALID;
  }
  const int g = std::max(1, std::min(LFM_AMAX_SLOTS, (cols + SPLITC_SC - 1) / SPLITC_SC));
  split16_cols_kernel<false><<<g, SPLITC_THREADS, 0, (cudaStream_t)stream>>>(src, rows, cols, cols_pad, part, cinv, hi, lo,
                                                                             ResIn());
  ++g_launches;
  return cuda_check(cudaGetLastError(), "split16_cols_kernel launch", err);
}

lfm_status k_split16_cols_residual(const float* Ax, const float* y, const float* w, const double* gamma, int cam,
                                   int rows, int cols, int cols_pad, float* part, float* cinv, uint16_t* hi, uint16_t* lo,
                                   void* stream, std::string& err) {
  if (cols % 4 || ((reinterpret_cast<uintptr_t>(Ax) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(w) |
                    reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo)) & 15)) {
    err = "split16_cols (residual): columns must be a multiple of 4 and rows 16-byte aligned";
    return LFM_E_INVALID;
  }
  ResIn ri;
  ri.Ax = Ax;
  ri.y = y;
  ri.w = w;
  ri.gamma = gamma;
  ri.cam = cam;
  const int g = std::max(1, std::min(LFM_AMAX_SLOTS, (cols + SPLITC_SC - 1) / SPLITC_SC));
  split16_cols_kernel<true><<<g, SPLITC_THREADS, 0, (cudaStream_t)stream>>>(nullptr, rows, cols, cols_pad, part, cinv, hi, lo, ri);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "split16_cols_kernel (residual) launch", err);
}

lfm_status k_split16_rows(const float* src, int rows, int len, float* part, float* rinv, uint16_t* hi, uint16_t* lo,
                          void* stream, std::string& err) {
  const int g = std::min(std::min(g_num_sms() * 2, LFM_AMAX_SLOTS), std::max(1, (rows + 15) / 16));
  split16_rows_kernel<<<g, 512, 0, (cudaStream_t)stream>>>(src, rows, len, part, rinv, hi, lo);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "split16_rows_kernel launch", err);
}

lfm_status k_split16(const float* src, long long n, const float* amax, uint16_t* hi, uint16_t* lo, void* stream,
                     std::string& err) {
  split16_kernel<<<(unsigned)std::min<long long>((n / 4 + 255) / 256 + 1, (long long)g_num_sms() * 8), 256, 0,
                   (cudaStream_t)stream>>>(src, n, amax, hi, lo);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "split16_kernel launch", err);
}

lfm_status launch_sep(const SepOp& op, const float* src, float* out, int b0, int n_out, int accumulate,
                      void* stream, std::string& err, int out_r0, int out_r1, int win_r0, int win_r1, int out_c0,
                      int out_c1, float* part, size_t part_bytes, F16Src h16) {
  if (n_out <= 0) return LFM_OK;
  SepArgs a;
  a.src = src;
  a.out = out;
  if (b0 < 0 || n_out < 0 || b0 + n_out > op.n_out) {
    err = "launch_sep: output range outside the op";
    return LFM_E_INVALID;
  }
  a.out_stride = op.out_stride ? op.out_stride : (long long)op.n_os * op.n_ot;
  a.src_pitch = op.src_pitch ? op.src_pitch : op.n_is;
  a.out_pitch = op.out_pitch ? op.out_pitch : op.n_os;
  a.t_foff = op.ft->d_foff;
  a.t_frow = reinterpret_cast<const int4*>(op.ft->d_frow);
  a.t_fw = reinterpret_cast<const float4*>(op.ft->d_fw);
  a.t_moff = op.mgrp == 8 ? op.ft->d_m8off : op.ft->d_moff;
  a.t_mseg = reinterpret_cast<const int4*>(op.mgrp == 8 ? op.ft->d_m8seg : op.ft->d_mseg);
  a.t_mw = op.mgrp == 8 ? op.ft->d_m8w : op.ft->d_mw;
  a.terms = op.d_terms;
  a.offs = op.d_offs + b0;
  a.s_g = reinterpret_cast<const int4*>(op.fs->d_g);
  a.s_gw = op.fs->d_gw;
  a.t_g = reinterpret_cast<const int4*>(op.ft->d_g);
  a.t_gw = op.ft->d_gw;
  a.fp_s = op.d_fp_s;
  a.fp_t = op.d_fp_t;
  a.s_ngroups = op.fs->n_groups;
  a.t_ngroups = op.ft->n_groups;
  a.ntx = op.ntx;
  a.nty = op.nty;
  a.n_os = op.n_os;
  a.n_ot = op.n_ot;
  a.n_is = op.n_is;
  a.n_it = op.n_it;
  a.fsp = op.fs_max + 1;
  a.ftm = op.ft_max;
  a.wsm = op.ws_max;
  a.wtm = op.wt_max;
  a.nb = op.nb;
  a.nbuf = op.nbuf;
  a.s_ident = op.s_ident;
  a.ug = op.s_ident && !op.stage;
  a.out_scale = op.out_scale;
  a.accumulate = accumulate;
  // output rows [out_r0, out_r1): whole tiles covering the range (rows of partial tiles are computed too)
  const int r1 = out_r1 < 0 ? op.n_ot : std::min(out_r1, op.n_ot);
  const int r0 = std::max(0, out_r0);
  if (r1 <= r0) return LFM_OK;
  a.ty0 = r0 / op.tt;
  const int nty = (r1 + op.tt - 1) / op.tt - a.ty0;
  a.win_r0 = std::max(0, win_r0);
  a.win_r1 = win_r1 < 0 ? op.n_it : std::min(win_r1, op.n_it);
  dim3 grid(op.ntx, nty, n_out);
  cudaStream_t s = (cudaStream_t)stream;
  if (op.tout && op.kind != 3 && op.kind != 5) {
    err = "transposed output needs the band_m or band_f kernel";
    return LFM_E_INVALID;
  }
  if (op.kind == 8) {
    // tcgen05 t pass (band_u.cuh): one table, one unit-scale term per output, normal output, 16-byte rows
    if (!op.ft->d_uoff || op.tout || n_out != 1) { err = "band_u: needs the tcgen05 form, one output, normal output"; return LFM_E_INVALID; }
    const Term& term = op.terms[op.offs[b0]];
    const float* base = src + term.src_off + (long long)a.win_r0 * a.src_pitch;
    const int win_rows = a.win_r1 - a.win_r0;
    if (win_rows <= 0) {  // empty source window: the output is zero (or unchanged)
      if (!accumulate)
        for (int r = r0; r < r1; ++r)
          if (cudaMemsetAsync(out + (long long)b0 * a.out_stride + (long long)r * a.out_pitch, 0, (size_t)op.n_os * 4, s) != cudaSuccess)
            return cuda_check(cudaGetLastError(), "band_u memset", err);
      return LFM_OK;
    }
    // column window [c0, c1): the 256-column tiles that meet it (columns of edge tiles outside it are computed too)
    const int cw0 = std::max(0, out_c0), cw1 = out_c1 < 0 ? op.n_os : std::min(out_c1, op.n_os);
    if (cw1 <= cw0) return LFM_OK;
    const int nt0 = cw0 / 256, nt1 = (cw1 + 255) / 256;
    const int n_mt_all = op.ft->u_ntiles;
    const int mt0 = op.ft->u_mode ? 0 : r0 / 128;
    const int n_mt_l = op.ft->u_mode ? n_mt_all : (r1 + 127) / 128 - mt0;
    // split-K when the window leaves most SMs idle (row / column shards of the multi-GPU partition): each item's
    // live blocks in ksplit chunks, partial outputs in `part`, summed in a fixed order (deterministic)
    int ksplit = 1;
    const int items0 = n_mt_l * (nt1 - nt0);
    const long long kc_rows = (long long)n_mt_all * 128;
    const float* ob = out + (long long)b0 * a.out_stride;
    if (part && !op.ft->u_mode && 2 * items0 <= g_num_sms() && !std::getenv("LFM_NO_SPLITK") && a.out_pitch % 4 == 0 &&
        op.n_os % 4 == 0 && ((uintptr_t)ob & 15) == 0 && ((uintptr_t)part & 15) == 0) {
      ksplit = std::min(4, g_num_sms() / std::max(1, items0));
      while (ksplit > 1 && (size_t)ksplit * kc_rows * a.out_pitch * 4 > part_bytes) --ksplit;
    }
    // 2xFP16 form when the caller passes the pre-split source (api.cu decides, f16_ok) and the plan has the images
    const bool f16 = h16.hi && op.ft->d_uh;
    CUtensorMap map, omap, lmap;
    lfm_status st;
    bool src3d = false;
    if (f16) {  // fp16 hi / lo maps of the source window, 64-column x 16-row boxes, 128-byte swizzle
      const long long wo = (long long)a.win_r0 * a.src_pitch + term.src_off;
      // one 8 KB 3D box per source part instead of four 2 KB boxes: the TMA unit's rate grows with the box
      // (tools/microbench/tma_rate.cu on B200: 82 vs 36 B/cycle/SM); forward t pass 64.5 -> 50.2 us, adjoint
      // 72.7 -> 62.5 us, 2500 -> 2748 pairs/s.  LFM_U_SRC3D=0 keeps the 2D boxes (A/B).
      static const bool src3d_env = !std::getenv("LFM_U_SRC3D") || std::atoi(std::getenv("LFM_U_SRC3D")) != 0;
      src3d = src3d_env && op.n_is % 256 == 0;  // every column group inside the row (no reads past a row's end)
      if (src3d) {  // (64 columns, rows, column groups of 64): the group stride (128 B) overlaps the row stride
        const long long d3[3] = {64, win_rows, op.n_is / 64}, s3[2] = {a.src_pitch * 2, 128};
        const int b3[3] = {64, 16, 4};
        if ((st = encode3(&map, h16.hi + wo, d3, s3, b3, CU_TENSOR_MAP_SWIZZLE_128B, err, true)) != LFM_OK ||
            (st = encode3(&lmap, h16.lo + wo, d3, s3, b3, CU_TENSOR_MAP_SWIZZLE_128B, err, true)) != LFM_OK)
          return st;
      } else if ((st = encode_map(&map, h16.hi + wo, op.n_is, win_rows, a.src_pitch, 64, 16, CU_TENSOR_MAP_SWIZZLE_128B, err, true)) != LFM_OK ||
          (st = encode_map(&lmap, h16.lo + wo, op.n_is, win_rows, a.src_pitch, 64, 16, CU_TENSOR_MAP_SWIZZLE_128B, err, true)) != LFM_OK)
        return st;
    } else {
      st = encode_map(&map, base, op.n_is, win_rows, a.src_pitch, 32, 16, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, err);
      if (st != LFM_OK) return st;
      lmap = map;
    }
    const bool out16 = f16 && h16.out_hi;
    CUtensorMap olmap;
    if (out16) {
      if (ksplit > 1 || accumulate) { err = "band_u: fp16 output without split-K or accumulation"; return LFM_E_INVALID; }
      const long long oo = (long long)b0 * a.out_stride;
      if ((st = encode_map(&omap, h16.out_hi + oo, op.n_os, op.n_ot, a.out_pitch, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B, err, true)) != LFM_OK ||
          (st = encode_map(&olmap, h16.out_lo + oo, op.n_os, op.n_ot, a.out_pitch, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B, err, true)) != LFM_OK)
        return st;
    } else if (ksplit > 1)
      st = encode_map(&omap, part, op.n_os, (int)(ksplit * kc_rows), a.out_pitch, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B, err);
    else
      st = encode_map(&omap, out + (long long)b0 * a.out_stride, op.n_os, op.n_ot, a.out_pitch, 32, 32,
                      CU_TENSOR_MAP_SWIZZLE_128B, err);
    if (st != LFM_OK) return st;
    static bool smem_set[LFM_MAX_DEV];
    const int dv = cur_dev();
    if (!smem_set[dv]) {
      if (cudaFuncSetAttribute(band_u_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM) != cudaSuccess ||
          cudaFuncSetAttribute(band_u_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM) != cudaSuccess ||
          cudaFuncSetAttribute(band_u_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM) != cudaSuccess ||
          cudaFuncSetAttribute(band_u_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM) != cudaSuccess ||
          cudaFuncSetAttribute(band_u_kernel<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM) != cudaSuccess)
        return cuda_check(cudaGetLastError(), "band_u smem attribute", err);
      smem_set[dv] = true;
    }
    UArgs u;
    const int n_mt = op.ft->u_ntiles;
    u.A = op.ft->d_ua;
    u.H = op.ft->d_uh;
    u.amax = h16.amax;
    u.n_amax = LFM_AMAX_SLOTS;
    u.amax_scale = h16.amax_scale;
    u.cinv = h16.cinv;
    u.src3d = src3d ? 1 : 0;
    if (u.cinv && !out16) { err = "band_u: per-column source scales need the fp16 output form"; return LFM_E_INVALID; }
    u.out_scale16 = h16.out_scale16;
    u.blk_off = op.ft->d_uoff + (size_t)term.t_tab * n_mt;
    u.blk_k0 = op.ft->d_uk0;
    u.out = out + (long long)b0 * a.out_stride;
    u.out_pitch = a.out_pitch;
    u.n_rows = op.n_ot;
    u.n_cols = op.n_os;
    u.mt0 = mt0;
    u.n_mt = n_mt_l;
    u.nt0 = nt0;
    u.n_nt = nt1 - nt0;
    u.ksplit = ksplit;
    u.kc_rows = (int)kc_rows;
    u.k_shift = a.win_r0;
    u.k_end = a.win_r1;
    u.windowed = a.win_r0 > 0 || a.win_r1 < op.n_it;
    u.group = op.stages > 0 ? op.stages : 4;
    if (f16) {  // 2xFP16: 3 MMAs per block instead of 6, so twice the blocks per drain (same MMAs per accumulator
                // chain, and a drain -- 128 KB of TMEM reads -- no longer outlasts the group's MMAs)
      static const int g16 = std::getenv("LFM_U16_GROUP") ? std::atoi(std::getenv("LFM_U16_GROUP")) : 0;
      u.group = g16 > 0 ? g16 : 2 * u.group;
    }
    u.scale = f16 ? (float)std::ldexp((double)(op.out_scale * term.scale), -op.ft->u_wexp) : op.out_scale * term.scale;
    u.accumulate = ksplit > 1 ? 0 : accumulate;
    u.tile_mode = op.ft->u_mode;
    u.tm_nz = op.ft->u_nz;
    if (u.tile_mode && (r0 != 0 || r1 != op.n_ot)) { err = "band_u: slice-pair tiles need the full output row range"; return LFM_E_INVALID; }
    const int grid_u = std::min(u.n_mt * u.n_nt * u.ksplit, g_num_sms());
    if (out16) band_u_kernel<false, true, true><<<grid_u, U_THREADS, U_SMEM, s>>>(map, omap, lmap, olmap, u);
    else if (f16) {
      if (ksplit > 1) band_u_kernel<true, true><<<grid_u, U_THREADS, U_SMEM, s>>>(map, omap, lmap, omap, u);
      else band_u_kernel<false, true><<<grid_u, U_THREADS, U_SMEM, s>>>(map, omap, lmap, omap, u);
    } else {
      if (ksplit > 1) band_u_kernel<true><<<grid_u, U_THREADS, U_SMEM, s>>>(map, omap, lmap, omap, u);
      else band_u_kernel<false><<<grid_u, U_THREADS, U_SMEM, s>>>(map, omap, lmap, omap, u);
    }
    ++g_launches;
    if (ksplit > 1) {
      const int sr0 = mt0 * 128, sr1 = std::min(op.n_ot, (mt0 + n_mt_l) * 128);
      const int sc0 = nt0 * 256, sc1 = std::min(op.n_os, nt1 * 256);
      const long long n = (long long)(sr1 - sr0) * ((sc1 - sc0) / 4);
      sum_chunks_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, s>>>(
          part, out + (long long)b0 * a.out_stride, a.out_pitch, sr0, sr1, sc0, sc1, ksplit, (int)kc_rows, accumulate);
      ++g_launches;
    }
    return cuda_check(cudaGetLastError(), "band_u_kernel launch", err);
  }
  if (op.kind == 5) {
    if (!op.ft->d_foff) { err = "band_f: t family has no flat MSEG form"; return LFM_E_INVALID; }
#define LFM_BF_CASE(TS_, TT_, NT_) \
    if (op.ts == TS_ && op.tt == TT_ && op.nt == NT_) return launch_band_f<TS_, TT_, NT_>(a, grid, s, err, op.stages, op.tout);
    LFM_BF_CASE(128, 32, 256)
    LFM_BF_CASE(128, 16, 128)
    LFM_BF_CASE(128, 8, 64)
    LFM_BF_CASE(64, 32, 128)
    LFM_BF_CASE(64, 16, 64)
#undef LFM_BF_CASE
    err = "unsupported band_f tile";
    return LFM_E_INVALID;
  }
  if (op.kind == 3) {
    // L2-gather t-pass over MSEG segments: identity s, no shared memory
    if (!(op.mgrp == 8 ? op.ft->d_m8off : op.ft->d_moff)) { err = "band_m: t family has no MSEG form"; return LFM_E_INVALID; }
    if (op.mgrp == 8) {
#define LFM_BM8_CASE(TS_, TT_, NT_) \
      if (op.ts == TS_ && op.tt == TT_ && op.nt == NT_) return launch_band_m8<TS_, TT_, NT_>(a, grid, s, err, op.stages, op.tout);
      LFM_BM8_CASE(128, 32, 128)
      LFM_BM8_CASE(128, 16, 64)
      LFM_BM8_CASE(128, 64, 256)
      LFM_BM8_CASE(64, 32, 64)
#undef LFM_BM8_CASE
      err = "unsupported band_m (8-row groups) tile";
      return LFM_E_INVALID;
    }
#define LFM_BM_CASE(TS_, TT_, NT_) \
    if (op.ts == TS_ && op.tt == TT_ && op.nt == NT_) return launch_band_m<TS_, TT_, NT_>(a, grid, s, err, op.stages, op.tout);
    LFM_BM_CASE(128, 32, 256)
    LFM_BM_CASE(128, 16, 128)
    LFM_BM_CASE(128, 8, 64)
    LFM_BM_CASE(64, 32, 128)
    LFM_BM_CASE(64, 16, 64)
    LFM_BM_CASE(32, 32, 64)
#undef LFM_BM_CASE
    err = "unsupported band_m tile";
    return LFM_E_INVALID;
  }
  const size_t smem = sep_smem(op, op.nb);
#define LFM_SEP_CASE(TS_, TT_, NT_)                                                              \
  if (op.ts == TS_ && op.tt == TT_) {                                                           \
    const int mode = op.s_ident ? (op.stage ? 2 : 3) : (op.stage ? 0 : 1);                      \
    switch (mode) {                                                                             \
      case 0: return launch_sep_t<TS_, TT_, NT_, 0>(a, grid, smem, s, err);                     \
      case 1: return launch_sep_t<TS_, TT_, NT_, 1>(a, grid, smem, s, err);                     \
      case 2: return launch_sep_t<TS_, TT_, NT_, 2>(a, grid, smem, s, err);                     \
      default: return launch_sep_t<TS_, TT_, NT_, 3>(a, grid, smem, s, err);                    \
    }                                                                                           \
  }
  LFM_SEP_CASE(128, 64, 256)
  LFM_SEP_CASE(128, 32, 256)
  LFM_SEP_CASE(64, 64, 128)
  LFM_SEP_CASE(64, 32, 128)
  LFM_SEP_CASE(32, 32, 64)
#undef LFM_SEP_CASE
  err = "unsupported sep tile";
  return LFM_E_INVALID;
}

// ------------------------------------------------------------------------------------------
// Shear pass: out[i] = sum_k w[line][k] * in[pos + mlo[line] + k along the pass axis].  3D grid: x tiles of 32
// threads (coalesced rows), y tiles of 8, z chunks of SH_ZC; each thread walks SH_ZC voxels along z with the
// table and data loads of all of them in flight together (the pass is latency-bound, 8 B of HBM per voxel).
template <int TAPS, int SH_ZC>
__global__ void __launch_bounds__(256) shear_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                    const int32_t* __restrict__ mlo, const float* __restrict__ w,
                                                    int axis, int nx, int ny, int nz, int accumulate) {
  const int ix = blockIdx.x * 32 + threadIdx.x, iy = blockIdx.y * 8 + threadIdx.y, z0 = blockIdx.z * SH_ZC;
  if (ix >= nx || iy >= ny) return;
  const size_t plane = (size_t)nx * ny;
  float res[SH_ZC];
  if (axis == 0) {
    // z pass: one line (x, y) per thread, so the shift and the weights are loaded once and the input column is
    // read as one sliding window of SH_ZC + TAPS - 1 values (each input value loaded once, not TAPS times)
    const int line = ix + nx * iy;
    const int m0 = __ldg(mlo + line);
    float wk[TAPS];
#pragma unroll
    for (int k = 0; k < TAPS; k += 4) {
      const float4 w4 = __ldg(reinterpret_cast<const float4*>(w + (size_t)line * TAPS + k));
      wk[k] = w4.x; wk[k + 1] = w4.y; wk[k + 2] = w4.z; wk[k + 3] = w4.w;
    }
    const float* col = in + (size_t)iy * nx + ix;
    float win[SH_ZC + TAPS - 1];
#pragma unroll
    for (int i = 0; i < SH_ZC + TAPS - 1; ++i) {
      const int j = z0 + m0 + i;
      win[i] = (j >= 0 && j < nz) ? __ldg(col + (size_t)j * plane) : 0.f;
    }
#pragma unroll
    for (int q = 0; q < SH_ZC; ++q) {
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < TAPS; ++k) acc = fmaf(wk[k], win[q + k], acc);
      res[q] = acc;
    }
  } else {
#pragma unroll
  for (int q = 0; q < SH_ZC; ++q) {
    const int iz = z0 + q;
    res[q] = 0.f;
    if (iz >= nz) continue;
    const size_t idx = (size_t)iz * plane + (size_t)iy * nx + ix;
    int line, pos, n;
    size_t stride;
    if (axis == 0) { line = ix + nx * iy; pos = iz; n = nz; stride = plane; }
    else if (axis == 1) { line = iy + ny * iz; pos = ix; n = nx; stride = 1; }
    else { line = ix + nx * iz; pos = iy; n = ny; stride = nx; }
    const int m0 = __ldg(mlo + line);
    const float* wl = w + (size_t)line * TAPS;
    const float* src = in + idx - (size_t)pos * stride;  // start of this voxel's line
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < TAPS; k += 4) {
      const float4 w4 = __ldg(reinterpret_cast<const float4*>(wl + k));
      const float wk[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = pos + m0 + k + t;
        if (j >= 0 && j < n) acc = fmaf(wk[t], __ldg(src + (size_t)j * stride), acc);
      }
    }
    res[q] = acc;
  }
  }
#pragma unroll
  for (int q = 0; q < SH_ZC; ++q) {
    const int iz = z0 + q;
    if (iz >= nz) break;
    const size_t idx = (size_t)iz * plane + (size_t)iy * nx + ix;
    out[idx] = accumulate ? out[idx] + res[q] : res[q];
  }
}

// y pass (axis 2, lines (x, z) along y, stride nx): like the z pass, a thread owns one line and walks YC
// consecutive y with a sliding window of YC + TAPS - 1 loads (each input value loaded once); lanes take consecutive
// x, so every load and store is a coalesced row.  Same ascending-tap FMA order as shear_kernel: bit-identical.
template <int TAPS, int YC>
__global__ void __launch_bounds__(256) shear_y_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                      const int32_t* __restrict__ mlo, const float* __restrict__ w,
                                                      int nx, int ny, int nz, int accumulate) {
  const int ix = blockIdx.x * 32 + threadIdx.x, iz = blockIdx.y * 8 + threadIdx.y, y0 = blockIdx.z * YC;
  if (ix >= nx || iz >= nz) return;
  const int line = ix + nx * iz;
  const int m0 = __ldg(mlo + line);
  float wk[TAPS];
#pragma unroll
  for (int k = 0; k < TAPS; k += 4) {
    const float4 w4 = __ldg(reinterpret_cast<const float4*>(w + (size_t)line * TAPS + k));
    wk[k] = w4.x; wk[k + 1] = w4.y; wk[k + 2] = w4.z; wk[k + 3] = w4.w;
  }
  const size_t base = (size_t)iz * nx * ny + ix;
  float win[YC + TAPS - 1];
#pragma unroll
  for (int i = 0; i < YC + TAPS - 1; ++i) {
    const int j = y0 + m0 + i;
    win[i] = (j >= 0 && j < ny) ? __ldg(in + base + (size_t)j * nx) : 0.f;
  }
#pragma unroll
  for (int q = 0; q < YC; ++q) {
    const int iy = y0 + q;
    if (iy >= ny) break;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < TAPS; ++k) acc = fmaf(wk[k], win[q + k], acc);
    float* o = out + base + (size_t)iy * nx;
    *o = accumulate ? *o + acc : acc;
  }
}

// x pass (axis 1, the line runs along the contiguous axis, one shift m0 and one weight row per line): each thread
// owns 4 consecutive x of one line, loads the aligned float4 window that covers them plus the taps
// (ceil((TAPS + 6) / 4) LDG.128 instead of 4 TAPS scalar loads) and stores one float4.  Same FMA order as
// shear_kernel (taps ascending; out-of-range taps contribute exact zeros), so the results are identical.
template <int TAPS, int ZC>
__global__ void __launch_bounds__(256) shear_x4_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                       const int32_t* __restrict__ mlo, const float* __restrict__ w,
                                                       int nx, int ny, int nz, int accumulate) {
  constexpr int NV4 = (TAPS + 6 + 3) / 4;
  const int x4 = 4 * (blockIdx.x * 32 + threadIdx.x), iy = blockIdx.y * 8 + threadIdx.y, z0 = blockIdx.z * ZC;
  if (x4 >= nx || iy >= ny) return;
#pragma unroll
  for (int q = 0; q < ZC; ++q) {
    const int iz = z0 + q;
    if (iz >= nz) break;
    const int line = iy + ny * iz;
    const int m0 = __ldg(mlo + line);
    const int a = x4 + (m0 & ~3), r = m0 & 3;  // aligned window start (floor) and offset in it
    const float* row = in + ((size_t)iz * ny + iy) * nx;
    float v[4 * NV4];
#pragma unroll
    for (int i = 0; i < NV4; ++i) {
      const int j = a + 4 * i;
      const float4 t = (j >= 0 && j < nx) ? __ldg(reinterpret_cast<const float4*>(row + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * i] = t.x; v[4 * i + 1] = t.y; v[4 * i + 2] = t.z; v[4 * i + 3] = t.w;
    }
    float u[TAPS + 3];
#pragma unroll
    for (int j = 0; j < TAPS + 3; ++j) u[j] = r == 0 ? v[j] : r == 1 ? v[j + 1] : r == 2 ? v[j + 2] : v[j + 3];
    float wk[TAPS];
#pragma unroll
    for (int k = 0; k < TAPS; k += 4) {
      const float4 w4 = __ldg(reinterpret_cast<const float4*>(w + (size_t)line * TAPS + k));
      wk[k] = w4.x; wk[k + 1] = w4.y; wk[k + 2] = w4.z; wk[k + 3] = w4.w;
    }
    float res[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < TAPS; ++k) acc = fmaf(wk[k], u[i + k], acc);
      res[i] = acc;
    }
    float4* o = reinterpret_cast<float4*>(out + ((size_t)iz * ny + iy) * nx + x4);
    float4 r4 = make_float4(res[0], res[1], res[2], res[3]);
    if (accumulate) {
      const float4 p = *o;
      r4.x += p.x; r4.y += p.y; r4.z += p.z; r4.w += p.w;
    }
    *o = r4;
  }
}

lfm_status launch_shear(const ShearPass& sp, int dir, const float* in, float* out, int nx, int ny, int nz,
                        int accumulate, void* stream, std::string& err) {
  // z chunk per thread: the z pass reads a sliding window of ZC + TAPS - 1 values per ZC outputs, so longer
  // chunks cut its re-reads and its block count (B200 bench: 16 -> +1.5 % pairs/s, 32 -> +1.3 %, the rotation
  // alone unchanged at ~20 us, so the gain is overlap with the other camera); the in-plane passes keep 8
  static const int zc_z = std::getenv("LFM_SH_ZC") ? std::atoi(std::getenv("LFM_SH_ZC")) : 16;
  const int zc = sp.axis == 0 && (zc_z == 16 || zc_z == 32) ? zc_z : 8;  // instantiated chunks only
  // LFM_SH_X4: 0 = scalar shear_kernel, 1 = x4 with 8 z per thread, 2 = 4 z, 3 = 16 z, 4 (default) = 2 z, 5 = 1 z
  // (B200, 128^3 yaw camera, rotation fwd per direction: scalar 20.5 us, 16 z 22.6, 8 z 16.4, 4 z 13.2, 2 z 12.6,
  // 1 z 12.4; bench 2081 / 2089 / 2141 / 2169 / 2183 / 2180 pairs/s)
  static const int x4_mode = std::getenv("LFM_SH_X4") ? std::atoi(std::getenv("LFM_SH_X4")) : 4;
  if (sp.axis == 1 && x4_mode > 0 && nx % 4 == 0 && ((uintptr_t)in & 15) == 0 && ((uintptr_t)out & 15) == 0) {
    const int zx = x4_mode == 2 ? 4 : x4_mode == 3 ? 16 : x4_mode == 4 ? 2 : x4_mode == 5 ? 1 : 8;
    dim3 grid4((nx / 4 + 31) / 32, (ny + 7) / 8, (nz + zx - 1) / zx), blk4(32, 8);
    cudaStream_t s4 = (cudaStream_t)stream;
#define LFM_SHX4(T, Z) shear_x4_kernel<T, Z><<<grid4, blk4, 0, s4>>>(in, out, sp.d_mlo[dir], sp.d_w[dir], nx, ny, nz, accumulate)
#define LFM_SHX4_T(Z) if (sp.taps == 4) LFM_SHX4(4, Z); else if (sp.taps == 8) LFM_SHX4(8, Z); else LFM_SHX4(16, Z)
    if (zx == 4) { LFM_SHX4_T(4); }
    else if (zx == 2) { LFM_SHX4_T(2); }
    else if (zx == 1) { LFM_SHX4_T(1); }
    else if (zx == 16) { LFM_SHX4_T(16); }
    else { LFM_SHX4_T(8); }
#undef LFM_SHX4_T
#undef LFM_SHX4
    ++g_launches;
    return cuda_check(cudaGetLastError(), "shear_x4_kernel launch", err);
  }
  if (sp.axis == 2 && !std::getenv("LFM_SH_Y_SCALAR")) {
    dim3 gy((nx + 31) / 32, (nz + 7) / 8, (ny + 15) / 16), by(32, 8);
    cudaStream_t sy = (cudaStream_t)stream;
    if (sp.taps == 4) shear_y_kernel<4, 16><<<gy, by, 0, sy>>>(in, out, sp.d_mlo[dir], sp.d_w[dir], nx, ny, nz, accumulate);
    else if (sp.taps == 8) shear_y_kernel<8, 16><<<gy, by, 0, sy>>>(in, out, sp.d_mlo[dir], sp.d_w[dir], nx, ny, nz, accumulate);
    else shear_y_kernel<16, 16><<<gy, by, 0, sy>>>(in, out, sp.d_mlo[dir], sp.d_w[dir], nx, ny, nz, accumulate);
    ++g_launches;
    return cuda_check(cudaGetLastError(), "shear_y_kernel launch", err);
  }
  dim3 grid((nx + 31) / 32, (ny + 7) / 8, (nz + zc - 1) / zc), blk(32, 8);
  cudaStream_t s = (cudaStream_t)stream;
#define LFM_SHEAR(T, Z) shear_kernel<T, Z><<<grid, blk, 0, s>>>(in, out, sp.d_mlo[dir], sp.d_w[dir], sp.axis, nx, ny, nz, accumulate)
  if (zc == 16) {
    if (sp.taps == 4) LFM_SHEAR(4, 16);
    else if (sp.taps == 8) LFM_SHEAR(8, 16);
    else LFM_SHEAR(16, 16);
  } else if (zc == 32) {
    if (sp.taps == 4) LFM_SHEAR(4, 32);
    else if (sp.taps == 8) LFM_SHEAR(8, 32);
    else LFM_SHEAR(16, 32);
  } else {
    if (sp.taps == 4) LFM_SHEAR(4, 8);
    else if (sp.taps == 8) LFM_SHEAR(8, 8);
    else LFM_SHEAR(16, 8);
  }
#undef LFM_SHEAR
  ++g_launches;
  return cuda_check(cudaGetLastError(), "shear_kernel launch", err);
}

// ------------------------------------------------------------------------------------------
// Elementwise helpers and deterministic fp64 reductions
__global__ void copy_scale_kernel(const float* __restrict__ in, float* __restrict__ out, long long n, float scale,
                                  int accumulate) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float v = scale * in[i];
    out[i] = accumulate ? out[i] + v : v;
  }
}

// float4 form (both pointers 16-byte aligned): the same per-element arithmetic, 4 elements per access; the
// n % 4 tail is done by the first threads
__global__ void copy_scale4_kernel(const float* __restrict__ in, float* __restrict__ out, long long n, float scale,
                                   int accumulate) {
  const long long n4 = n >> 2, stride = (long long)gridDim.x * blockDim.x;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = t; i < n4; i += stride) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(in) + i);
    float4 v = make_float4(scale * a.x, scale * a.y, scale * a.z, scale * a.w);
    if (accumulate) {
      const float4 o = reinterpret_cast<const float4*>(out)[i];
      v.x = o.x + v.x; v.y = o.y + v.y; v.z = o.z + v.z; v.w = o.w + v.w;
    }
    reinterpret_cast<float4*>(out)[i] = v;
  }
  if (t < (n & 3)) {
    const long long i = 4 * n4 + t;
    const float v = scale * in[i];
    out[i] = accumulate ? out[i] + v : v;
  }
}

__global__ void fill_kernel(float* __restrict__ out, long long n, float v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = v;
}

__global__ void mul_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                           long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}

constexpr int RED_BLOCKS = 1184;  // 8 x 148 SMs (partials: 3 x 1184 doubles fit the workspace's 16384)
constexpr int STATS_BLOCKS = 592; // 4 x 148: the stats kernel's blocks all resident at once (64 registers x 256)
constexpr int RED_THREADS = 256;

__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NV>
__device__ inline void block_sum_store(double (&v)[NV], double* part) {
  __shared__ double sh[NV][RED_THREADS / 32];
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) sh[q][wid] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0;
      for (int w = 0; w < RED_THREADS / 32; ++w) s += sh[q][w];
      part[(size_t)blockIdx.x * NV + q] = s;
    }
  }
}

// stats: [sum w y Ax, sum w y y, sum w Ax Ax] (fp64 products and sums; float4 loads when the three vectors are
// 16-byte aligned, the n % 4 tail by the first threads)
template <bool VEC>
__global__ void __launch_bounds__(RED_THREADS, STATS_BLOCKS / 148) stats_partial_kernel(const float* __restrict__ Ax,
                                                                    const float* __restrict__ y,
                                                                    const float* __restrict__ w, long long n,
                                                                    double* part) {
  double v[3] = {0, 0, 0};
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x, stride = (long long)gridDim.x * blockDim.x;
  auto acc = [&](double a, double yy, double ww) {
    v[0] += ww * yy * a;
    v[1] += ww * yy * yy;
    v[2] += ww * a * a;
  };
  long long i0 = t;
  if (VEC) {
    // LD float4 of each vector per iteration: 3 LD 16-byte loads in flight before the fp64 sums need them; LD = 2
    // keeps the kernel at 64 registers, so all STATS_BLOCKS (4 per SM) are resident in one wave (with LD = 4 it took
    // 124 registers: 2 blocks per SM, two waves)
    constexpr int LD = 2;
    const long long n4 = n >> 2;
    const float4* A4 = reinterpret_cast<const float4*>(Ax);
    const float4* Y4 = reinterpret_cast<const float4*>(y);
    const float4* W4 = reinterpret_cast<const float4*>(w);
    for (long long i = t; i < n4; i += LD * stride) {  // every lane's LD x 3 loads issued before any sum
      float4 a[LD], b[LD], c[LD];
#pragma unroll
      for (int j = 0; j < LD; ++j) {
        const long long k = i + j * stride;
        const bool ok = k < n4;
        a[j] = ok ? __ldg(A4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
        b[j] = ok ? __ldg(Y4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
        c[j] = ok ? __ldg(W4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < LD; ++j)
        if (i + j * stride < n4) {
          acc(a[j].x, b[j].x, c[j].x); acc(a[j].y, b[j].y, c[j].y); acc(a[j].z, b[j].z, c[j].z); acc(a[j].w, b[j].w, c[j].w);
        }
    }
    i0 = 4 * n4 + t;
  }
  for (long long i = i0; i < n; i += stride) acc(Ax[i], y[i], w[i]);
  block_sum_store<3>(v, part);
}

// final sum of nblocks block partials per value: one block of 256 threads per value q, thread t adds the partials
// b = t, t + 256, ... in order, then a fixed-shape tree -- the same order every run (deterministic), and the
// partial loads are spread over 256 threads instead of one dependent chain
__global__ void __launch_bounds__(256) reduce_final_kernel(const double* __restrict__ part, int nblocks, int nv,
                                                           double* out, int accumulate) {
  __shared__ double sh[256];
  const int q = blockIdx.x, t = threadIdx.x;
  double s = 0;
#pragma unroll 8
  for (int b = t; b < nblocks; b += 256) s += part[(size_t)b * nv + q];
  sh[t] = s;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (t < h) sh[t] += sh[t + h];
    __syncthreads();
  }
  if (t == 0) out[q] = accumulate ? out[q] + sh[0] : sh[0];
}

__global__ void gains_kernel(const double* __restrict__ stats, int n_cam, double* gamma, int* flag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int bad = 0;
  gamma[0] = 1.0;
  for (int c = 1; c < n_cam; ++c) {
    double num = stats[3 * c], den = stats[3 * c + 1];
    if (!(den > 0.0)) { bad = 1; gamma[c] = 0.0; }
    else gamma[c] = num / den;
  }
  if (flag) *flag = bad;
}

// r = w (Ax - gamma y); partial 1/2 sum w (Ax - gamma y)^2 (COST only); float4 form when aligned
template <bool VEC, bool COST>
__global__ void __launch_bounds__(RED_THREADS) residual_kernel(const float* __restrict__ Ax, const float* __restrict__ y,
                                                               const float* __restrict__ w,
                                                               const double* __restrict__ gamma, int cam,
                                                               float* __restrict__ r, long long n, double* part) {
  const float g = (float)gamma[cam];
  double v[1] = {0};
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x, stride = (long long)gridDim.x * blockDim.x;
  auto one = [&](float a, float b, float c) {
    const float d = a - g * b;
    if (COST) v[0] += 0.5 * (double)c * (double)d * (double)d;
    return c * d;
  };
  long long i0 = t;
  if (VEC) {
    const long long n4 = n >> 2;
    for (long long i = t; i < n4; i += stride) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(Ax) + i);
      const float4 b = __ldg(reinterpret_cast<const float4*>(y) + i);
      const float4 c = __ldg(reinterpret_cast<const float4*>(w) + i);
      const float r0 = one(a.x, b.x, c.x), r1 = one(a.y, b.y, c.y), r2 = one(a.z, b.z, c.z), r3 = one(a.w, b.w, c.w);
      reinterpret_cast<float4*>(r)[i] = make_float4(r0, r1, r2, r3);
    }
    i0 = 4 * n4 + t;
  }
  for (long long i = i0; i < n; i += stride) r[i] = one(Ax[i], y[i], w[i]);
  if (COST) block_sum_store<1>(v, part);
}

// grad += beta * sum_{l in N_j, in grid} (x_j - x_l) + nu;  partial [nu*x_j + (beta/4) sum_l (x_j-x_l)^2] (COST)
// Tiled: a block of 32 x 8 threads owns 32 x 8 (x, y) columns and a chunk of R26_ZC slices; the R26_ZC + 2 planes
// of the (32+2) x (16+2) footprint are loaded into shared memory at once (every load in flight together, one
// barrier; x is read from HBM/L2 about 1.4 times).  Each thread walks its column up the chunk keeping the 3 x 3
// neighbourhoods of planes z-1, z, z+1 in registers, so every shared value is loaded once per plane (9 loads per
// voxel instead of 26).  Neighbours outside the grid contribute nothing: their shared values are 0, so their terms
// are x_j, taken back out after the sum (n_out x_j); the sum runs in the order dz, dy, dx ascending.
constexpr int R26_ZC = 16, R26_TY = 8, R26_NT = 32 * R26_TY;
// VEC (nx % 4 == 0): the footprint rows are loaded as 10 aligned float4 [x0 - 4, x0 + 36) (16-byte cp.async, whole
// float4s in or out of the grid), so the load loop issues 1800 instead of 6120 copies per block with cheaper index
// arithmetic -- the kernel is issue-bound (ncu: 79 % issue-active, integer pipe 65 %), not DRAM-bound.
template <bool COST, bool VEC>
__global__ void __launch_bounds__(R26_NT) reg26_kernel(const float* __restrict__ x, float* __restrict__ grad, int nx,
                                                    int ny, int nz, float beta, float nu, double* part) {
  constexpr int PX = VEC ? 40 : 34, XO = VEC ? 3 : 0, PY = R26_TY + 2, PP = PX * PY;
  __shared__ __align__(16) float pl[R26_ZC + 2][PY][PX];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * R26_TY, z0 = blockIdx.z * R26_ZC;
  const int ix = x0 + tx, iy = y0 + ty;
  const size_t plane = (size_t)nx * ny;
  if constexpr (VEC) {
    constexpr int NV = (R26_ZC + 2) * PY * 10;  // float4 per block
    for (int e = tid; e < NV; e += R26_NT) {
      const int row = e / 10, lv = e - row * 10;  // row = pz * PY + ly
      const int pz = row / PY, ly = row - pz * PY;
      const int gx = x0 - 4 + 4 * lv, gy = y0 + ly - 1, zz = z0 + pz - 1;
      const bool ok = zz >= 0 && zz < nz && gy >= 0 && gy < ny && gx >= 0 && gx < nx;
      const float* src = ok ? x + (size_t)zz * plane + (size_t)gy * nx + gx : x;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(&pl[0][0][0] + 4 * e)),
                   "l"(src), "r"(ok ? 16 : 0) : "memory");
    }
  } else {
    constexpr int NE = (R26_ZC + 2) * PP;
    // the footprint straight into shared memory (cp.async, 4 bytes; zero-filled outside the grid): every load in
    // flight at once without holding registers, so two blocks fit an SM and one's loads overlap the other's sums
    for (int e = tid; e < NE; e += R26_NT) {
      const int pz = e / PP, r = e - pz * PP, ly = r / PX, lx = r - ly * PX;
      const int gx = x0 + lx - 1, gy = y0 + ly - 1, zz = z0 + pz - 1;
      const bool ok = zz >= 0 && zz < nz && gx >= 0 && gx < nx && gy >= 0 && gy < ny;
      const float* src = ok ? x + (size_t)zz * plane + (size_t)gy * nx + gx : x;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(&pl[0][0][0] + e)),
                   "l"(src), "r"(ok ? 4 : 0) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int cxy = (1 + (ix > 0) + (ix < nx - 1)) * (1 + (iy > 0) + (iy < ny - 1));  // in-grid x, y neighbours (+self)
  double v = 0;
  if (ix < nx && iy < ny) {
    // the chunk's grad values loaded together (read-modify-write: one latency for the chunk, not one per voxel)
    float gin[R26_ZC];
#pragma unroll
    for (int q = 0; q < R26_ZC; ++q)
      gin[q] = z0 + q < nz ? grad[(size_t)(z0 + q) * plane + (size_t)iy * nx + ix] : 0.f;
    if constexpr (VEC && !COST) {
      // gradient only (the FISTA loop): sum_{l in N_j} (x_j - x_l) = n_in x_j - sum_{l in N_j} x_l, with the
      // neighbour sum taken as 3 x 3 plane sums that slide along z (each plane summed once, not three times) and
      // the out-of-grid neighbours zero in the footprint: (27 - n_out) x_j - (S_{z-1} + S_z + S_{z+1}).  About a
      // third of the instructions of the literal 26-difference order (which the cost path keeps); the two differ
      // by fp32 summation order only.
      float S[3], xc[3];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        float r[3];
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
          r[dy] = (pl[d][ty + dy][tx + XO] + pl[d][ty + dy][tx + XO + 1]) + pl[d][ty + dy][tx + XO + 2];
        S[d] = (r[0] + r[1]) + r[2];
        xc[d] = pl[d][ty + 1][tx + XO + 1];
      }
#pragma unroll
      for (int q = 0; q < R26_ZC; ++q) {
        const int iz = z0 + q;
        if (iz >= nz) break;
        {
          float r[3];
#pragma unroll
          for (int dy = 0; dy < 3; ++dy)
            r[dy] = (pl[q + 2][ty + dy][tx + XO] + pl[q + 2][ty + dy][tx + XO + 1]) + pl[q + 2][ty + dy][tx + XO + 2];
          S[(q + 2) % 3] = (r[0] + r[1]) + r[2];
          xc[(q + 2) % 3] = pl[q + 2][ty + 1][tx + XO + 1];
        }
        const float xj = xc[(q + 1) % 3];
        const int n_out = 27 - (1 + (iz > 0) + (iz < nz - 1)) * cxy;
        const float g = (float)(27 - n_out) * xj - ((S[q % 3] + S[(q + 1) % 3]) + S[(q + 2) % 3]);
        grad[(size_t)iz * plane + (size_t)iy * nx + ix] = gin[q] + (beta * g + nu);
      }
    } else {
    float P[3][9];  // 3 x 3 neighbourhoods of planes q, q+1, q+2 (z-1, z, z+1) of the footprint
#pragma unroll
    for (int d = 0; d < 2; ++d)
#pragma unroll
      for (int k = 0; k < 9; ++k) P[d][k] = pl[d][ty + k / 3][tx + XO + k % 3];
#pragma unroll
    for (int q = 0; q < R26_ZC; ++q) {
      const int iz = z0 + q;
      if (iz >= nz) break;
#pragma unroll
      for (int k = 0; k < 9; ++k) P[(q + 2) % 3][k] = pl[q + 2][ty + k / 3][tx + XO + k % 3];
      const float xj = P[(q + 1) % 3][4];
      // all 26 differences in the order dz, dy, dx (outside the grid the shared value is 0, so such a term is x_j);
      // the n_out of them are taken back out after the sum (interior voxels: n_out = 0, the plain sum)
      float g = 0.f;
      double rs = 0;
#pragma unroll
      for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
            if (dz == 1 && dy == 1 && dx == 1) continue;
            const float d = xj - P[(q + dz) % 3][dy * 3 + dx];
            g += d;
            if (COST) rs += (double)d * (double)d;
          }
      const int n_out = 27 - (1 + (iz > 0) + (iz < nz - 1)) * cxy;
      if (n_out) {
        g -= (float)n_out * xj;
        if (COST) rs -= (double)n_out * (double)xj * (double)xj;
      }
      const size_t i = (size_t)iz * plane + (size_t)iy * nx + ix;
      grad[i] = gin[q] + (beta * g + nu);
      if (COST) v += (double)nu * xj + 0.25 * (double)beta * rs;
    }
    }
  }
  if (COST) {
    // block partial (R26_TY warps), fixed order
    __shared__ double sh[R26_TY];
    const double a = warp_sum(v);
    if (tx == 0) sh[ty] = a;
    __syncthreads();
    if (tid == 0) {
      double t = 0;
      for (int w = 0; w < R26_TY; ++w) t += sh[w];
      part[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
  }
}

__global__ void fista_kernel(float* __restrict__ x, float* __restrict__ z, const float* __restrict__ grad,
                             const float* __restrict__ d, long long n, float tau) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float xn = fmaxf(0.f, z[i] - grad[i] / d[i]);
    z[i] = xn + tau * (xn - x[i]);
    x[i] = xn;
  }
}

// float4 form (all four vectors 16-byte aligned): the same per-element arithmetic, the n % 4 tail by the first threads
__device__ __forceinline__ void fista_one(float& xv, float& zv, float gv, float dv, float tau) {
  const float xn = fmaxf(0.f, zv - gv / dv);
  zv = xn + tau * (xn - xv);
  xv = xn;
}
__global__ void fista4_kernel(float* __restrict__ x, float* __restrict__ z, const float* __restrict__ grad,
                              const float* __restrict__ d, long long n, float tau) {
  const long long n4 = n >> 2, stride = (long long)gridDim.x * blockDim.x;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = t; i < n4; i += stride) {
    float4 xv = reinterpret_cast<float4*>(x)[i], zv = reinterpret_cast<float4*>(z)[i];
    const float4 gv = __ldg(reinterpret_cast<const float4*>(grad) + i), dv = __ldg(reinterpret_cast<const float4*>(d) + i);
    fista_one(xv.x, zv.x, gv.x, dv.x, tau);
    fista_one(xv.y, zv.y, gv.y, dv.y, tau);
    fista_one(xv.z, zv.z, gv.z, dv.z, tau);
    fista_one(xv.w, zv.w, gv.w, dv.w, tau);
    reinterpret_cast<float4*>(x)[i] = xv;
    reinterpret_cast<float4*>(z)[i] = zv;
  }
  for (long long i = 4 * n4 + t; i < n; i += stride) fista_one(x[i], z[i], grad[i], d[i], tau);
}

__global__ void majoriser_finish_kernel(float* __restrict__ d, long long n, float add) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = fmaxf(d[i] + add, 1e-12f);
}

static unsigned ew_grid(long long n) { return (unsigned)std::min<long long>((n + 255) / 256, 148 * 16); }

lfm_status k_copy_scale(const float* in, float* out, long long n, float scale, int acc, void* s, std::string& err) {
  if ((((uintptr_t)in | (uintptr_t)out) & 15) == 0)
    copy_scale4_kernel<<<ew_grid((n + 3) / 4), 256, 0, (cudaStream_t)s>>>(in, out, n, scale, acc);
  else
    copy_scale_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)s>>>(in, out, n, scale, acc);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "copy_scale", err);
}
lfm_status k_fill(float* out, long long n, float v, void* s, std::string& err) {
  fill_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)s>>>(out, n, v);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "fill", err);
}
lfm_status k_mul(const float* a, const float* b, float* out, long long n, void* s, std::string& err) {
  mul_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)s>>>(a, b, out, n);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "mul", err);
}
static bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

lfm_status k_stats(const float* Ax, const float* y, const float* w, long long n, double* part, double* out, void* s,
                   std::string& err) {
  if (al16(Ax) && al16(y) && al16(w))
    stats_partial_kernel<true><<<STATS_BLOCKS, RED_THREADS, 0, (cudaStream_t)s>>>(Ax, y, w, n, part);
  else
    stats_partial_kernel<false><<<STATS_BLOCKS, RED_THREADS, 0, (cudaStream_t)s>>>(Ax, y, w, n, part);
  reduce_final_kernel<<<3, 256, 0, (cudaStream_t)s>>>(part, STATS_BLOCKS, 3, out, 0);
  g_launches += 2;
  return cuda_check(cudaGetLastError(), "stats", err);
}
lfm_status k_gains(const double* stats, int n_cam, double* gamma, int* flag, void* s, std::string& err) {
  gains_kernel<<<1, 32, 0, (cudaStream_t)s>>>(stats, n_cam, gamma, flag);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "gains", err);
}
lfm_status k_residual(const float* Ax, const float* y, const float* w, const double* gamma, int cam, float* r,
                      long long n, double* part, double* cost, int cost_acc, void* s, std::string& err) {
  const bool vec = al16(Ax) && al16(y) && al16(w) && al16(r);
  cudaStream_t st = (cudaStream_t)s;
  if (cost) {
    if (vec) residual_kernel<true, true><<<RED_BLOCKS, RED_THREADS, 0, st>>>(Ax, y, w, gamma, cam, r, n, part);
    else residual_kernel<false, true><<<RED_BLOCKS, RED_THREADS, 0, st>>>(Ax, y, w, gamma, cam, r, n, part);
    reduce_final_kernel<<<1, 256, 0, st>>>(part, RED_BLOCKS, 1, cost, cost_acc);
    g_launches += 2;
  } else {
    if (vec) residual_kernel<true, false><<<ew_grid((n + 3) / 4), RED_THREADS, 0, st>>>(Ax, y, w, gamma, cam, r, n, nullptr);
    else residual_kernel<false, false><<<ew_grid(n), RED_THREADS, 0, st>>>(Ax, y, w, gamma, cam, r, n, nullptr);
    ++g_launches;
  }
  return cuda_check(cudaGetLastError(), "residual", err);
}
lfm_status k_reg26(const float* x, float* grad, int nx, int ny, int nz, float beta, float nu, double* part,
                   double* cost, void* s, std::string& err) {
  dim3 grid((nx + 31) / 32, (ny + R26_TY - 1) / R26_TY, (nz + R26_ZC - 1) / R26_ZC), blk(32, R26_TY);
  const long long nblk = (long long)grid.x * grid.y * grid.z;
  if (cost && nblk > 4096 * 4) { err = "reg26: volume too large for the reduction partials"; return LFM_E_INVALID; }
  const bool vec = nx % 4 == 0 && ((uintptr_t)x & 15) == 0 && !std::getenv("LFM_R26_SCALAR");
  if (cost) {
    if (vec) reg26_kernel<true, true><<<grid, blk, 0, (cudaStream_t)s>>>(x, grad, nx, ny, nz, beta, nu, part);
    else reg26_kernel<true, false><<<grid, blk, 0, (cudaStream_t)s>>>(x, grad, nx, ny, nz, beta, nu, part);
    reduce_final_kernel<<<1, 256, 0, (cudaStream_t)s>>>(part, (int)nblk, 1, cost, 0);
    g_launches += 2;
  } else {
    if (vec) reg26_kernel<false, true><<<grid, blk, 0, (cudaStream_t)s>>>(x, grad, nx, ny, nz, beta, nu, nullptr);
    else reg26_kernel<false, false><<<grid, blk, 0, (cudaStream_t)s>>>(x, grad, nx, ny, nz, beta, nu, nullptr);
    ++g_launches;
  }
  return cuda_check(cudaGetLastError(), "reg26", err);
}
lfm_status k_fista(float* x, float* z, const float* grad, const float* d, long long n, float tau, void* s,
                   std::string& err) {
  if (al16(x) && al16(z) && al16(grad) && al16(d))
    fista4_kernel<<<ew_grid((n + 3) / 4), 256, 0, (cudaStream_t)s>>>(x, z, grad, d, n, tau);
  else
    fista_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)s>>>(x, z, grad, d, n, tau);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "fista", err);
}
lfm_status k_majoriser_finish(float* d, long long n, float add, void* s, std::string& err) {
  majoriser_finish_kernel<<<ew_grid(n), 256, 0, (cudaStream_t)s>>>(d, n, add);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "majoriser_finish", err);
}

}  // namespace lfm

namespace lfm {
// ------------------------------------------------------------------------------------------
// Plan-time autotuning (host side of plan creation, excluded from timed work): every hot op of
// A_forward / A_adjoint times each shared-memory-feasible (tile, threads, staging, nb) candidate on
// zero-filled scratch buffers with CUDA events and keeps the fastest.  It runs only with LFM_AUTOTUNE=1; the
// default is the fixed tcgen05 choice of tc_defaults (no timed launches at plan creation).
static void free_sep_dev(SepOp& op) {
  dfree(op.d_terms); dfree(op.d_offs); dfree(op.d_fp_s); dfree(op.d_fp_t);
  op.d_terms = nullptr; op.d_offs = nullptr; op.d_fp_s = nullptr; op.d_fp_t = nullptr;
}

// Optional result cache (LFM_TUNE_FILE): lines "<key> <op> ts tt nt nb stage"; a hit skips the timing
// (used so that ncu captures see only the measured launches).
static std::string tune_key(const CameraPlan& cp) {
  // field by field (struct padding never enters the hash), plus the rotated voxel sizes, which fix every band
  unsigned long long h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  const lfm_camera& c = cp.cam;
  const int iv[] = {c.type, c.basis, c.k_s, c.k_t, c.nl_s, c.nl_t, c.n_a, c.n_s, c.n_t};
  const double dv[] = {c.f_main, c.ap_s, c.ap_t, c.d_scene, c.d_det, c.d_mu_m, c.d_d_mu, c.f_mu, c.fill, c.px_s, c.px_t};
  mix(iv, sizeof(iv));
  mix(dv, sizeof(dv));
  mix(c.R, sizeof(c.R));
  mix(cp.info.vox_r, sizeof(cp.info.vox_r));
  char buf[96];
  // v7: keyed field by field with the rotated voxel sizes
  std::snprintf(buf, sizeof(buf), "v7_%016llx_%dx%dx%d", h, cp.info.nx, cp.info.ny, cp.info.nz);
  return buf;
}

// Overrides and layout conditions applied to whichever choice was made (timed or default):
// LFM_FWD_T / LFM_ADJ_T = 0 direct sep, 1 transpose + band_m/band_f, 2 direct s-pass kernels, 3 band_v.
static void finish_choice(CameraPlan& cp, bool dbg, float t_x, float t_z) {
  if (const char* e = std::getenv("LFM_FWD_T")) cp.fwd_t = e[0] - '0';
  if (const char* e = std::getenv("LFM_ADJ_T")) cp.adj_t = e[0] - '0';
  if (cp.fwd_t == 1 && !(cp.fwd_p1.fs && (cp.fwd_p1.kind == 3 || cp.fwd_p1.kind == 5))) cp.fwd_t = 0;
  if (cp.adj_t == 1 && !(cp.adj_a2.fs && (cp.adj_a2.kind == 3 || cp.adj_a2.kind == 5))) cp.adj_t = 0;
  // band_v moves rows by TMA: 16-byte row strides of the volume and of the detector intermediates
  const bool tc_ok = cp.info.nx % 4 == 0 && cp.adj_c1.n_os % 4 == 0 && cp.cf[0].n_rows % 4 == 0;
  if (cp.fwd_t == 3 && !tc_ok) cp.fwd_t = 2;
  if (cp.adj_t == 3 && !tc_ok) cp.adj_t = 2;
  if (cp.fwd_t < 0 || cp.fwd_t > 3) cp.fwd_t = 0;
  if (cp.adj_t < 0 || cp.adj_t > 3) cp.adj_t = 0;
  if (const char* fs = std::getenv("LFM_FWD_SPLIT")) cp.fwd_split = fs[0] == '1';
  static const char* smode[] = {"direct sep", "transposed", "spass", "tcgen05"};
  if (dbg)
    std::fprintf(stderr, "[lfm] collapsed forward: %s, s pass %s (transpose x %.3f, z %.3f ms x2); adjoint s pass %s\n",
                 cp.fwd_split ? "two passes" : "fused", smode[cp.fwd_t], t_x, t_z, smode[cp.adj_t]);
}

// B200 default (no timing, LFM_AUTOTUNE unset or 0): the collapsed path in its two-pass form with the tcgen05
// kernels wherever their layout conditions hold -- band_u for both t passes (fwd_c2, adj_c1; drain group 4)
// and band_v for both s passes -- the choice the timed search makes on B200 at 64^3-256^3.
// The other ops keep the cost model's tiles.  LFM_FORCE_<op> still wins.
static lfm_status tc_defaults(CameraPlan& cp, std::string& err) {
  std::vector<std::pair<SepOp*, const char*>> ops = {{&cp.fwd_c2, "fwd_c2"}, {&cp.adj_c1, "adj_c1"}};
  for (Component& cm : cp.comps) {
    ops.push_back({&cm.fwd_c2, "fwd_c2"});
    ops.push_back({&cm.adj_c1, "adj_c1"});
  }
  for (auto pr : ops) {
    SepOp& op = *pr.first;
    if (!op.fs || std::getenv((std::string("LFM_FORCE_") + pr.second).c_str())) continue;
    const long long sp = op.src_pitch ? op.src_pitch : op.n_is;
    if (op.ft->u_off.empty() || op.tout || op.n_out != 1 || op.terms.size() != 1 || (sp & 3) ||
        (op.terms[0].src_off & 3) || std::getenv("LFM_NO_TC"))
      continue;
    op.kind = 8; op.ts = 256; op.tt = 128; op.nt = U_THREADS; op.nb = 1; op.stage = 0; op.stages = 4; op.mgrp = 4;
    fill_sep_geometry(op);
    free_sep_dev(op);
    size_t bytes = 0;
    lfm_status st = upload_sep(op, bytes, err);
    if (st != LFM_OK) return st;
  }
  cp.fwd_split = 1;
  cp.fwd_t = std::getenv("LFM_NO_VF") ? 2 : 3;
  cp.adj_t = std::getenv("LFM_NO_VA") ? 2 : 3;
  return LFM_OK;
}

lfm_status autotune_camera(CameraPlan& cp, std::string& err) {
  const char* env = std::getenv("LFM_AUTOTUNE");
  if (!env || env[0] != '1' || !cp.comps.empty()) {  // non-separable lenslet stages: the tcgen05 defaults
    lfm_status st = tc_defaults(cp, err);
    finish_choice(cp, std::getenv("LFM_DEBUG") != nullptr, -1.f, -1.f);
    return st;
  }
  const char* tfile = std::getenv("LFM_TUNE_FILE");
  const std::string key = tune_key(cp);
  std::vector<std::string> cached;
  if (tfile) {
    if (FILE* f = std::fopen(tfile, "r")) {
      char line[256];
      while (std::fgets(line, sizeof(line), f)) cached.push_back(line);
      std::fclose(f);
    }
  }
  SepOp* ops[] = {&cp.fwd_s1, &cp.fwd_s3, &cp.adj_s3, &cp.adj_s1, &cp.fwd_c, &cp.adj_c1, &cp.adj_c2,
                  &cp.fwd_c1, &cp.fwd_c2, &cp.fwd_p1, &cp.adj_a2};
  const char* names[] = {"fwd_s1", "fwd_s3", "adj_s3", "adj_s1", "fwd_c", "adj_c1", "adj_c2", "fwd_c1", "fwd_c2",
                         "fwd_p1", "adj_a2"};
  constexpr int NQ_OPS = 11;
  float op_best[NQ_OPS];
  for (float& v : op_best) v = -1.f;
  const bool dbg = std::getenv("LFM_DEBUG") != nullptr;
  const bool dbg_all = std::getenv("LFM_DEBUG_TUNE") != nullptr;  // every candidate's time
  size_t src_n = 0, out_n = 0;
  for (SepOp* op : ops) {
    if (!op->fs) continue;
    long long mx = 0;
    for (const Term& t : op->terms) mx = std::max(mx, t.src_off);
    const long long sp = op->src_pitch ? op->src_pitch : op->n_is;
    const long long opch = op->out_pitch ? op->out_pitch : op->n_os;
    const long long ost = op->out_stride ? op->out_stride : (long long)op->n_os * op->n_ot;
    const long long nr = op->tout ? op->n_os : op->n_ot, nc = op->tout ? op->n_ot : op->n_os;
    src_n = std::max(src_n, (size_t)(mx + (long long)(op->n_it - 1) * sp + op->n_is + 16));
    out_n = std::max(out_n, (size_t)((long long)(std::min(op->n_out, 64) - 1) * ost + (nr - 1) * opch + nc + 16));
  }
  float *src = nullptr, *out = nullptr;
  if (cudaMalloc(&src, src_n * 4) != cudaSuccess || cudaMalloc(&out, out_n * 4) != cudaSuccess) {
    cudaGetLastError();
    dfree(src);
    if (dbg) std::fprintf(stderr, "[lfm] autotune skipped: no scratch memory\n");
    return LFM_OK;
  }
  cudaMemset(src, 0, src_n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int cand[][3] = {{128, 64, 256}, {128, 32, 256}, {64, 64, 128}, {64, 32, 128}, {32, 32, 64}};
  lfm_status st = LFM_OK;
  for (int q = 0; q < NQ_OPS && st == LFM_OK; ++q) {
    SepOp& op = *ops[q];
    if (!op.fs) continue;
    if (std::getenv((std::string("LFM_FORCE_") + names[q]).c_str())) continue;  // explicit override wins
    bool hit = false;
    for (const std::string& ln : cached) {
      char k[128], o[32];
      int ts, tt, nt, nb, stg;
      int kind = 0, stages = 2;
      float ms = 0;
      int mg = 4, chk = 32;
      if (std::sscanf(ln.c_str(), "%127s %31s %d %d %d %d %d %d %d %f %d %d", k, o, &ts, &tt, &nt, &nb, &stg, &kind,
                      &stages, &ms, &mg, &chk) == 12 &&
          key == k && std::string(o) == names[q]) {
        op.ts = ts; op.tt = tt; op.nt = nt; op.nb = nb; op.stage = stg; op.kind = kind; op.stages = stages; op.mgrp = mg;
        op.chunk = chk;
        op_best[q] = ms;
        fill_sep_geometry(op);
        free_sep_dev(op);
        size_t bytes = 0;
        if ((st = upload_sep(op, bytes, err)) != LFM_OK) break;
        hit = true;
      }
    }
    if (hit || st != LFM_OK) continue;
    const int n_out = std::min(op.n_out, 64);
    const SepOp keep = op;  // cost-model choice (device pointers of `op` are replaced below)
    int bts = keep.ts, btt = keep.tt, bnt = keep.nt, bnb = keep.nb, bst = keep.stage;
    float best = 1e30f;
    int bkind = keep.kind, bstages = keep.stages, bmgrp = keep.mgrp, bchunk = keep.chunk;
    if (op.s_ident && (op.n_is % 4) == 0) {
      op.kind = 0;
      const int mcand[][4] = {{128, 32, 256, 4}, {128, 16, 128, 4}, {128, 8, 64, 4},  {64, 32, 128, 4},
                              {64, 16, 64, 4},   {32, 32, 64, 4},   {128, 32, 128, 8}, {128, 16, 64, 8},
                              {128, 64, 256, 8}, {64, 32, 64, 8}};
      for (auto& c : mcand) {
        if (st != LFM_OK || !op.ft->want_mseg) break;
        if (c[3] == 8 && op.ft->m8_off.empty()) continue;
        bool aligned = true;
        for (const Term& t : op.terms) aligned &= (t.src_off % 4) == 0;
        if (!aligned) break;
        for (int unr : {4, 8}) {
          op.kind = 3; op.ts = c[0]; op.tt = c[1]; op.nt = c[2]; op.nb = 1; op.stage = 0; op.stages = unr; op.mgrp = c[3];
          fill_sep_geometry(op);
          free_sep_dev(op);
          size_t bytes = 0;
          if ((st = upload_sep(op, bytes, err)) != LFM_OK) break;
          float ms = 0, tot = 0;
          bool ok = true;
          for (int rep = 0; rep < 3 && ok; ++rep) {
            cudaEventRecord(e0, 0);
            ok = launch_sep(op, src, out, 0, n_out, 0, nullptr, err) == LFM_OK;
            cudaEventRecord(e1, 0);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0) tot += ms;
          }
          if (!ok || cudaGetLastError() != cudaSuccess) continue;
          if (dbg_all)
            std::fprintf(stderr, "[lfm]   %-7s band_m %3dx%-3d nt %3d unroll %d grp %d: %.3f ms\n", names[q], c[0], c[1], c[2],
                         unr, c[3], tot / 2);
          if (tot < best) { best = tot; bts = c[0]; btt = c[1]; bnt = c[2]; bnb = 1; bst = 0; bkind = 3; bstages = unr; bmgrp = c[3]; }
        }
      }
      op.kind = 0;
      const int fcand[][3] = {{128, 32, 256}, {128, 16, 128}, {128, 8, 64}, {64, 32, 128}, {64, 16, 64}};
      for (auto& c : fcand) {
        if (st != LFM_OK || !op.ft->want_mseg) break;
        bool aligned = true;
        for (const Term& t : op.terms) aligned &= (t.src_off % 4) == 0;
        if (!aligned) break;
        for (int unr : {1, 2}) {
          op.kind = 5; op.ts = c[0]; op.tt = c[1]; op.nt = c[2]; op.nb = 1; op.stage = 0; op.stages = unr; op.mgrp = 4;
          fill_sep_geometry(op);
          free_sep_dev(op);
          size_t bytes = 0;
          if ((st = upload_sep(op, bytes, err)) != LFM_OK) break;
          float ms = 0, tot = 0;
          bool ok = true;
          for (int rep = 0; rep < 3 && ok; ++rep) {
            cudaEventRecord(e0, 0);
            ok = launch_sep(op, src, out, 0, n_out, 0, nullptr, err) == LFM_OK;
            cudaEventRecord(e1, 0);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0) tot += ms;
          }
          if (!ok || cudaGetLastError() != cudaSuccess) continue;
          if (dbg_all)
            std::fprintf(stderr, "[lfm]   %-7s band_f %3dx%-3d nt %3d unroll %d: %.3f ms\n", names[q], c[0], c[1], c[2], unr,
                         tot / 2);
          if (tot < best) { best = tot; bts = c[0]; btt = c[1]; bnt = c[2]; bnb = 1; bst = 0; bkind = 5; bstages = unr; bmgrp = 4; }
        }
      }
      op.kind = 0;
      // band_u: tcgen05 (one output, one term, normal output, 16-byte source rows); stages = drain group
      for (int grp : {4, 8}) {
        const long long sp = op.src_pitch ? op.src_pitch : op.n_is;
        if (st != LFM_OK || op.ft->u_off.empty() || op.tout || op.n_out != 1 || op.terms.size() != 1 ||
            (sp & 3) || (op.terms[0].src_off & 3) || std::getenv("LFM_NO_TC"))
          break;
        op.kind = 8; op.ts = 256; op.tt = 128; op.nt = U_THREADS; op.nb = 1; op.stage = 0; op.stages = grp; op.mgrp = 4;
        fill_sep_geometry(op);
        free_sep_dev(op);
        size_t bytes = 0;
        if ((st = upload_sep(op, bytes, err)) != LFM_OK) break;
        float ms = 0, tot = 0;
        bool ok = true;
        for (int rep = 0; rep < 3 && ok; ++rep) {
          cudaEventRecord(e0, 0);
          ok = launch_sep(op, src, out, 0, n_out, 0, nullptr, err) == LFM_OK;
          cudaEventRecord(e1, 0);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep > 0) tot += ms;
        }
        if (!ok || cudaGetLastError() != cudaSuccess) continue;
        if (dbg_all) std::fprintf(stderr, "[lfm]   %-7s band_u group %d: %.3f ms\n", names[q], grp, tot / 2);
        // the second drain group must win by 2 % (ties otherwise flip between runs)
        if (tot < (grp == 4 ? best : 0.98f * best)) { best = tot; bts = 256; btt = 128; bnt = U_THREADS; bnb = 1; bst = 0; bkind = 8; bstages = grp; bmgrp = 4; }
      }
      op.kind = 0;
    }
    for (auto& c : cand) {
      if (op.tout) break;
      for (int stage : {1, 0}) {
        for (int nb : {1, 2, 4}) {
          if (nb > 1 && op.terms.size() < (size_t)op.n_out * 2) continue;
          op.ts = c[0]; op.tt = c[1]; op.nt = c[2]; op.stage = stage; op.nb = nb;
          fill_sep_geometry(op);
          if (sep_smem(op, nb) > (size_t)210 * 1024) continue;
          free_sep_dev(op);
          size_t bytes = 0;
          if ((st = upload_sep(op, bytes, err)) != LFM_OK) break;
          float ms = 0, tot = 0;
          bool ok = true;
          for (int rep = 0; rep < 3 && ok; ++rep) {
            cudaEventRecord(e0, 0);
            ok = launch_sep(op, src, out, 0, n_out, 0, nullptr, err) == LFM_OK;
            cudaEventRecord(e1, 0);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0) tot += ms;
          }
          if (!ok || cudaGetLastError() != cudaSuccess) continue;
          if (tot < best) { best = tot; bts = c[0]; btt = c[1]; bnt = c[2]; bnb = nb; bst = stage; bkind = 0; }
        }
        if (st != LFM_OK) break;
      }
      if (st != LFM_OK) break;
    }
    op.ts = bts; op.tt = btt; op.nt = bnt; op.nb = bnb; op.stage = bst; op.kind = bkind; op.stages = bstages; op.mgrp = bmgrp;
    op.chunk = bchunk;
    fill_sep_geometry(op);
    free_sep_dev(op);
    size_t bytes = 0;
    if (st == LFM_OK) st = upload_sep(op, bytes, err);
    op_best[q] = best * (float)op.n_out / (float)n_out;  // per launch over all outputs
    if (dbg)
      std::fprintf(stderr, "[lfm] autotune %-7s -> %s tile %3dx%-3d nt %3d nb %d stage %d stages %d grp %d (%.3f ms for %d outputs)\n",
                   names[q], op.kind == 3 ? "band_m" : op.kind == 5 ? "band_f" : op.kind == 8 ? "band_u" : "sep   ", op.ts, op.tt, op.nt, op.nb, op.stage, op.stages, op.mgrp, best / 2, n_out);
    if (tfile && st == LFM_OK) {
      if (FILE* f = std::fopen(tfile, "a")) {
        std::fprintf(f, "%s %s %d %d %d %d %d %d %d %.6f %d %d\n", key.c_str(), names[q], op.ts, op.tt, op.nt, op.nb,
                     op.stage, op.kind, op.stages, op_best[q], op.mgrp, op.chunk);
        std::fclose(f);
      }
    }
  }
  // s passes of the two-pass path: direct (sep kernel) or transpose + band_m with transposed output
  float t_x = -1.f, t_z = -1.f;
  int cached_decision[3] = {-1, -1, -1};
  for (const std::string& ln : cached) {
    char k[128], o[32];
    int d0, d1, d2;
    if (std::sscanf(ln.c_str(), "%127s %31s %d %d %d", k, o, &d0, &d1, &d2) == 5 && key == k && std::string(o) == "decide") {
      cached_decision[0] = d0; cached_decision[1] = d1; cached_decision[2] = d2;
    }
  }
  if (st == LFM_OK && cached_decision[0] < 0 && (op_best[9] > 0 || op_best[10] > 0)) {
    const int nx = cp.info.nx, ny = cp.info.ny, nz = cp.info.nz, nd = cp.adj_c1.n_os;
    const long long nslice = (long long)nx * ny;
    auto time_it = [&](auto&& fn) {
      float ms = 0, tot = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0, 0);
        fn();
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0) tot += ms;
      }
      return tot;
    };
    std::string terr;
    t_x = time_it([&] { k_transpose(src, out, nz, ny, nx, nslice, nx, nslice, ny, nullptr, terr); });
    t_z = time_it([&] {
      k_transpose(src, out, nz, ny, nd, nd, (long long)nz * nd, (long long)nd * ny, ny, nullptr, terr);
    });
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  dfree(src);
  dfree(out);
  if (op_best[9] > 0 && op_best[7] > 0 && t_x >= 0) cp.fwd_t = (t_x + op_best[9]) < op_best[7];
  if (op_best[10] > 0 && op_best[6] > 0 && t_z >= 0) cp.adj_t = (t_z + op_best[10]) < op_best[6];
  // transposed output exists only in band_m / band_f
  cp.fwd_t = cp.fwd_t && cp.fwd_p1.fs && (cp.fwd_p1.kind == 3 || cp.fwd_p1.kind == 5);
  cp.adj_t = cp.adj_t && cp.adj_a2.fs && (cp.adj_a2.kind == 3 || cp.adj_a2.kind == 5);
  float fwd_s = cp.fwd_t ? t_x + op_best[9] : op_best[7];
  // direct s passes (spass.cuh, mode 2): timed against the choice above, kept when faster
  if (st == LFM_OK && cached_decision[0] < 0) {
    float* sb = nullptr;
    float* ob = nullptr;
    const size_t big = std::max((size_t)cp.info.ny * cp.info.nz * cp.adj_c1.n_os, (size_t)cp.info.n_vox) * 4;
    if (cudaMalloc(&sb, big) == cudaSuccess && cudaMalloc(&ob, big) == cudaSuccess) {
      cudaMemset(sb, 0, big);
      cudaEvent_t f0, f1;
      cudaEventCreate(&f0);
      cudaEventCreate(&f1);
      auto time2 = [&](auto&& fn) {
        float ms = 0, tot = 0;
        bool ok = true;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(f0, 0);
          ok &= fn() == LFM_OK;
          cudaEventRecord(f1, 0);
          cudaEventSynchronize(f1);
          cudaEventElapsedTime(&ms, f0, f1);
          if (rep > 0) tot += ms;
        }
        return ok ? tot : -1.f;
      };
      std::string terr;
      const float t_sf = time2([&] { return k_spass_fwd(cp, sb, ob, nullptr, terr); });
      cp.spa_vta = 4;
      const float t_sa4 = time2([&] { return k_spass_adj(cp, sb, ob, 0, nullptr, terr); });
      cp.spa_vta = 8;
      const float t_sa8 = time2([&] { return k_spass_adj(cp, sb, ob, 0, nullptr, terr); });
      cp.spa_vta = (t_sa4 > 0 && (t_sa8 <= 0 || t_sa4 < t_sa8)) ? 4 : 8;
      const float t_sa = cp.spa_vta == 4 ? t_sa4 : t_sa8;
      float adj_s = cp.adj_t ? t_z + op_best[10] : op_best[6];
      const float t_vf = std::getenv("LFM_NO_VF") ? -1.f : time2([&] { return k_vpass_fwd(cp, cp.vf, sb, ob, nullptr, terr); });
      const float t_va = std::getenv("LFM_NO_VA") ? -1.f : time2([&] { return k_vpass_adj(cp, cp.va, sb, ob, 0, nullptr, terr); });
      if (dbg)
        std::fprintf(stderr, "[lfm] direct s passes: fwd %.3f / tc %.3f ms (vs %.3f), adj %.3f / tc %.3f ms (vs %.3f) x2\n",
                     t_sf, t_vf, fwd_s, t_sa, t_va, adj_s);
      if (t_sf > 0 && (fwd_s <= 0 || t_sf < fwd_s)) { cp.fwd_t = 2; fwd_s = t_sf; }
      if (t_sa > 0 && (adj_s <= 0 || t_sa < adj_s)) { cp.adj_t = 2; adj_s = t_sa; }
      if (t_vf > 0 && (fwd_s <= 0 || t_vf < fwd_s)) { cp.fwd_t = 3; fwd_s = t_vf; }
      if (t_va > 0 && (adj_s <= 0 || t_va < adj_s)) { cp.adj_t = 3; adj_s = t_va; }
      cudaEventDestroy(f0);
      cudaEventDestroy(f1);
    }
    cudaGetLastError();
    dfree(sb);
    dfree(ob);
  }
  // forward order: fused (fwd_c) or two passes (s pass + fwd_c2), whichever timed faster
  if (cached_decision[0] < 0 && op_best[4] > 0 && fwd_s > 0 && op_best[8] > 0) cp.fwd_split = (fwd_s + op_best[8]) < op_best[4];
  if (cached_decision[0] >= 0) {
    cp.fwd_split = cached_decision[0];
    cp.fwd_t = cached_decision[1];
    cp.adj_t = cached_decision[2];
  } else if (tfile) {
    if (FILE* f = std::fopen(tfile, "a")) {
      std::fprintf(f, "%s decide %d %d %d\n", key.c_str(), cp.fwd_split, cp.fwd_t, cp.adj_t);
      std::fclose(f);
    }
  }
  finish_choice(cp, dbg, t_x, t_z);
  return st;
}
}  // namespace lfm
