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
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "lfm_internal.h"
#include "lfm_kernels.h"

namespace lfm {

thread_local int g_launches = 0;

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

static lfm_status upload_family(BandFamily& f, size_t& bytes, std::string& err) {
  if (f.n_tables == 0) return LFM_OK;
  std::vector<float> w32(f.ew64.size());
  for (size_t i = 0; i < w32.size(); ++i) w32[i] = (float)f.ew64[i];  // one rounding fp64 -> fp32
  lfm_status st = dev_upload(&f.d_cnt, f.cnt.data(), f.cnt.size() * sizeof(int32_t), err);
  if (st != LFM_OK) return st;
  if ((st = dev_upload(&f.d_idx, f.eidx.data(), f.eidx.size() * sizeof(int32_t), err)) != LFM_OK) return st;
  bytes += f.cnt.size() * 4 + f.eidx.size() * 4 + w32.size() * 4;
  return dev_upload(&f.d_w, w32.data(), w32.size() * sizeof(float), err);
}

static void footprints(const BandFamily& f, int tile, std::vector<Footprint>& fp, int& ntiles) {
  ntiles = (f.n_rows + tile - 1) / tile;
  fp.assign((size_t)f.n_tables * ntiles, Footprint{0, 0});
  for (int m = 0; m < f.n_tables; ++m)
    for (int t = 0; t < ntiles; ++t) {
      int lo, w;
      ell_footprint(f, m, tile, t, lo, w);
      fp[(size_t)m * ntiles + t] = Footprint{lo, w};
    }
}

static lfm_status upload_sep(SepOp& op, size_t& bytes, std::string& err) {
  if (!op.fs) return LFM_OK;
  lfm_status st = dev_upload(&op.d_terms, op.terms.data(), op.terms.size() * sizeof(Term), err);
  if (st != LFM_OK) return st;
  st = dev_upload(&op.d_offs, op.offs.data(), op.offs.size() * sizeof(int32_t), err);
  if (st != LFM_OK) return st;
  std::vector<Footprint> fs, ft;
  footprints(*op.fs, op.ts, fs, op.ntx);
  footprints(*op.ft, op.tt, ft, op.nty);
  st = dev_upload(&op.d_fp_s, fs.data(), fs.size() * sizeof(Footprint), err);
  if (st != LFM_OK) return st;
  bytes += op.terms.size() * sizeof(Term) + (fs.size() + ft.size()) * sizeof(Footprint);
  return dev_upload(&op.d_fp_t, ft.data(), ft.size() * sizeof(Footprint), err);
}

lfm_status upload_camera(CameraPlan& cp, std::string& err) {
  size_t bytes = 0;
  lfm_status st;
  for (int ax = 0; ax < 2; ++ax) {
    BandFamily* fams[] = {&cp.s1f[ax], &cp.s1a[ax], &cp.s3f[ax], &cp.s3a[ax], &cp.cf[ax], &cp.ca[ax]};
    for (BandFamily* f : fams)
      if ((st = upload_family(*f, bytes, err)) != LFM_OK) return st;
  }
  for (BandFamily* f : {&cp.id_s, &cp.id_t, &cp.id_vt})
    if ((st = upload_family(*f, bytes, err)) != LFM_OK) return st;
  SepOp* ops[] = {&cp.fwd_s1, &cp.fwd_s3, &cp.adj_s3, &cp.adj_s1, &cp.fwd_c, &cp.adj_c1, &cp.adj_c2,
                  &cp.xp_s1f, &cp.xp_s1a, &cp.xp_s3f, &cp.xp_s3a};
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
  cp.info.table_bytes = bytes;
  return LFM_OK;
}

static void dfree(void* p) {
  if (p) cudaFree(p);
}

void free_camera(CameraPlan& cp) {
  std::vector<BandFamily*> fams = {&cp.id_s, &cp.id_t, &cp.id_vt};
  for (int ax = 0; ax < 2; ++ax)
    for (BandFamily* f : {&cp.s1f[ax], &cp.s1a[ax], &cp.s3f[ax], &cp.s3a[ax], &cp.cf[ax], &cp.ca[ax]})
      fams.push_back(f);
  for (BandFamily* f : fams) {
    dfree(f->d_cnt); dfree(f->d_idx); dfree(f->d_w);
    f->d_cnt = nullptr; f->d_idx = nullptr; f->d_w = nullptr;
  }
  SepOp* ops[] = {&cp.fwd_s1, &cp.fwd_s3, &cp.adj_s3, &cp.adj_s1, &cp.fwd_c, &cp.adj_c1, &cp.adj_c2,
                  &cp.xp_s1f, &cp.xp_s1a, &cp.xp_s3f, &cp.xp_s3a};
  for (SepOp* op : ops) {
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
// Separable banded sum (ELL tables)
struct SepArgs {
  const float* src;
  float* out;
  long long out_stride;
  const Term* terms;
  const int32_t* offs;  // already offset by b0
  const int32_t* s_cnt;
  const int32_t* s_idx;
  const float* s_w;
  const int32_t* t_cnt;
  const int32_t* t_idx;
  const float* t_w;
  const Footprint* fp_s;
  const Footprint* fp_t;
  int s_ell, t_ell;
  int ntx, nty;
  int n_os, n_ot, n_is, n_it;
  int fsp;   // smem row pitch of the staged source / T1 tiles
  int ftm;   // max staged rows
  float out_scale;
  int accumulate;
};

constexpr int SEP_THREADS = 256;

// TAPS_S > 0: s entries held in registers (<= TAPS_S per row); TAPS_S == 0: runtime loop from L1.
template <int TS, int TT, int TAPS_S>
__global__ void __launch_bounds__(SEP_THREADS) sep_kernel(SepArgs a) {
  extern __shared__ float smem[];
  constexpr int ROW_STEP = SEP_THREADS / TS;       // rows between a thread's outputs
  constexpr int R = TS * TT / SEP_THREADS;          // outputs per thread
  static_assert(R >= 1 && TS * TT % SEP_THREADS == 0, "tile must be a multiple of the block");
  const int tid = threadIdx.x;
  const int tx = blockIdx.x, ty = blockIdx.y, b = blockIdx.z;
  const int os0 = tx * TS, ot0 = ty * TT;
  float* stage = smem;                               // [ftm][fsp]
  float* t1 = stage + (size_t)a.ftm * a.fsp;         // [TT][fsp]
  float* tw = t1 + (size_t)TT * a.fsp;               // [TT][t_ell]
  int* tix = (int*)(tw + TT * a.t_ell);              // [TT][t_ell]
  int* tcn = tix + TT * a.t_ell;                     // [TT]
  // zero-fill once so padded (zero-weight) taps only ever read finite values
  for (int e = tid; e < (a.ftm + TT) * a.fsp; e += SEP_THREADS) smem[e] = 0.f;

  const int my_s = tid % TS;
  const int my_t0 = tid / TS;
  const int os = os0 + my_s;
  const bool s_ok = os < a.n_os;
  float acc[R], acc_hi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { acc[r] = 0.f; acc_hi[r] = 0.f; }

  const int e0 = a.offs[b], e1 = a.offs[b + 1];
  int since_flush = 0;
  for (int e = e0; e < e1; ++e) {
    const Term term = a.terms[e];
    const Footprint fs = a.fp_s[(size_t)term.s_tab * a.ntx + tx];
    const Footprint ft = a.fp_t[(size_t)term.t_tab * a.nty + ty];
    if (fs.width == 0 || ft.width == 0) continue;    // CTA-uniform: no contribution to this tile
    __syncthreads();                                  // previous term finished with smem
    const float* src = a.src + term.src_off;
    // stage the source footprint rows [ft.lo, ft.lo+ft.width) x cols [fs.lo, fs.lo+fs.width)
    const int nst = ft.width * fs.width;
    for (int q = tid; q < nst; q += SEP_THREADS) {
      int r = q / fs.width, c = q - r * fs.width;
      int row = ft.lo + r, col = fs.lo + c;
      float v = 0.f;
      if (row < a.n_it && col < a.n_is) v = __ldg(src + (size_t)row * a.n_is + col);
      stage[r * a.fsp + c] = v;
    }
    // this tile's t-rows: counts, footprint-relative source rows, weights
    {
      const size_t tb = (size_t)term.t_tab * a.t_ell * a.n_ot;
      for (int q = tid; q < TT * a.t_ell; q += SEP_THREADS) {
        int tt = q / a.t_ell, k = q - tt * a.t_ell;
        int row = ot0 + tt;
        float w = 0.f;
        int ix = 0;
        if (row < a.n_ot) {
          w = __ldg(a.t_w + tb + (size_t)k * a.n_ot + row);
          ix = min(max(__ldg(a.t_idx + tb + (size_t)k * a.n_ot + row) - ft.lo, 0), ft.width - 1);
        }
        tw[q] = w;
        tix[q] = ix;
      }
      for (int tt = tid; tt < TT; tt += SEP_THREADS) {
        int row = ot0 + tt;
        tcn[tt] = row < a.n_ot ? __ldg(a.t_cnt + (size_t)term.t_tab * a.n_ot + row) : 0;
      }
    }
    __syncthreads();
    // t-pass (minor direction first): t1[tt][c] = sum_k tw[tt][k] * stage[tix[tt][k]][c]
    const int nt1 = TT * fs.width;
    for (int q = tid; q < nt1; q += SEP_THREADS) {
      int tt = q / fs.width, c = q - tt * fs.width;
      const float* wr = tw + tt * a.t_ell;
      const int* ir = tix + tt * a.t_ell;
      const int cn = tcn[tt];
      float v = 0.f;
      for (int k = 0; k < cn; ++k) v = fmaf(wr[k], stage[ir[k] * a.fsp + c], v);
      t1[tt * a.fsp + c] = v;
    }
    __syncthreads();
    // s-pass: my column os, rows my_t0 + r*ROW_STEP, exact non-zero list (padded to the warp max)
    {
      const size_t sb = (size_t)term.s_tab * a.s_ell * a.n_os;
      const int cnt = s_ok ? __ldg(a.s_cnt + (size_t)term.s_tab * a.n_os + os) : 0;
      const int cmax = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
      if constexpr (TAPS_S > 0) {
        float w[TAPS_S];
        int ix[TAPS_S];
#pragma unroll
        for (int k = 0; k < TAPS_S; ++k) {
          w[k] = 0.f;
          ix[k] = 0;
          if (k < cmax && s_ok) {
            w[k] = __ldg(a.s_w + sb + (size_t)k * a.n_os + os) * term.scale;
            ix[k] = min(max(__ldg(a.s_idx + sb + (size_t)k * a.n_os + os) - fs.lo, 0), fs.width - 1);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float* tr = t1 + (my_t0 + r * ROW_STEP) * a.fsp;
          float v = 0.f;
#pragma unroll
          for (int k = 0; k < TAPS_S; ++k)
            if (k < cmax) v = fmaf(w[k], tr[ix[k]], v);
          acc[r] += v;
        }
      } else {
        for (int k = 0; k < cmax; ++k) {
          float wk = 0.f;
          int ik = 0;
          if (s_ok) {
            wk = __ldg(a.s_w + sb + (size_t)k * a.n_os + os) * term.scale;
            ik = min(max(__ldg(a.s_idx + sb + (size_t)k * a.n_os + os) - fs.lo, 0), fs.width - 1);
          }
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fmaf(wk, t1[(my_t0 + r * ROW_STEP) * a.fsp + ik], acc[r]);
        }
      }
    }
    if (++since_flush == 16) {  // blocked accumulation (keeps long positive sums accurate)
#pragma unroll
      for (int r = 0; r < R; ++r) { acc_hi[r] += acc[r]; acc[r] = 0.f; }
      since_flush = 0;
    }
  }
  if (!s_ok) return;
  float* outb = a.out + (size_t)b * a.out_stride;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int row = ot0 + my_t0 + r * ROW_STEP;
    if (row >= a.n_ot) continue;
    float v = a.out_scale * (acc_hi[r] + acc[r]);
    float* p = outb + (size_t)row * a.n_os + os;
    *p = a.accumulate ? *p + v : v;
  }
}

template <int TS, int TT, int TAPS_S>
static lfm_status launch_sep_t(const SepArgs& a, dim3 grid, size_t smem, cudaStream_t s, std::string& err) {
  auto kern = sep_kernel<TS, TT, TAPS_S>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(sep_kernel)", err);
    configured = true;
  }
  kern<<<grid, SEP_THREADS, smem, s>>>(a);
  ++g_launches;
  return cuda_check(cudaGetLastError(), "sep_kernel launch", err);
}

template <int TS, int TT>
static lfm_status launch_sep_taps(const SepArgs& a, dim3 grid, size_t smem, cudaStream_t s, std::string& err) {
  if (a.s_ell <= 4) return launch_sep_t<TS, TT, 4>(a, grid, smem, s, err);
  if (a.s_ell <= 8) return launch_sep_t<TS, TT, 8>(a, grid, smem, s, err);
  if (a.s_ell <= 16) return launch_sep_t<TS, TT, 16>(a, grid, smem, s, err);
  return launch_sep_t<TS, TT, 0>(a, grid, smem, s, err);
}

lfm_status launch_sep(const SepOp& op, const float* src, float* out, int b0, int n_out, int accumulate,
                      void* stream, std::string& err) {
  if (n_out <= 0) return LFM_OK;
  SepArgs a;
  a.src = src;
  a.out = out;
  a.out_stride = (long long)op.n_os * op.n_ot;
  a.terms = op.d_terms;
  a.offs = op.d_offs + b0;
  a.s_cnt = op.fs->d_cnt;
  a.s_idx = op.fs->d_idx;
  a.s_w = op.fs->d_w;
  a.t_cnt = op.ft->d_cnt;
  a.t_idx = op.ft->d_idx;
  a.t_w = op.ft->d_w;
  a.fp_s = op.d_fp_s;
  a.fp_t = op.d_fp_t;
  a.s_ell = op.fs->ell;
  a.t_ell = op.ft->ell;
  a.ntx = op.ntx;
  a.nty = op.nty;
  a.n_os = op.n_os;
  a.n_ot = op.n_ot;
  a.n_is = op.n_is;
  a.n_it = op.n_it;
  a.fsp = op.fs_max + 1;  // +1: odd pitch spreads t-pass rows over banks
  a.ftm = op.ft_max;
  a.out_scale = op.out_scale;
  a.accumulate = accumulate;
  size_t smem = ((size_t)a.ftm * a.fsp + (size_t)op.tt * a.fsp) * 4 + (size_t)op.tt * a.t_ell * 8 + (size_t)op.tt * 4;
  dim3 grid(op.ntx, op.nty, n_out);
  cudaStream_t s = (cudaStream_t)stream;
  const int ts = op.ts, tt = op.tt;
  if (ts == 64 && tt == 32) return launch_sep_taps<64, 32>(a, grid, smem, s, err);
  if (ts == 64 && tt == 16) return launch_sep_taps<64, 16>(a, grid, smem, s, err);
  if (ts == 32 && tt == 32) return launch_sep_taps<32, 32>(a, grid, smem, s, err);
  if (ts == 32 && tt == 16) return launch_sep_taps<32, 16>(a, grid, smem, s, err);
  if (ts == 16 && tt == 16) return launch_sep_taps<16, 16>(a, grid, smem, s, err);
  err = "unsupported sep tile";
  return LFM_E_INVALID;
}

// ------------------------------------------------------------------------------------------
// Shear pass: out[i] = sum_k w[line][k] * in[pos + mlo[line] + k along the pass axis]
template <int TAPS>
__global__ void __launch_bounds__(256) shear_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                    const int32_t* __restrict__ mlo, const float* __restrict__ w,
                                                    int axis, int nx, int ny, int nz, int accumulate) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long nvox = (long long)nx * ny * nz;
  if (idx >= nvox) return;
  int ix = (int)(idx % nx);
  long long r = idx / nx;
  int iy = (int)(r % ny);
  int iz = (int)(r / ny);
  int line, pos, n;
  long long stride;
  if (axis == 0) { line = ix + nx * iy; pos = iz; n = nz; stride = (long long)nx * ny; }
  else if (axis == 1) { line = iy + ny * iz; pos = ix; n = nx; stride = 1; }
  else { line = ix + nx * iz; pos = iy; n = ny; stride = nx; }
  const int m0 = __ldg(mlo + line);
  const float* wl = w + (size_t)line * TAPS;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < TAPS; k += 4) {
    float4 w4 = __ldg(reinterpret_cast<const float4*>(wl + k));
    float wk[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int j = pos + m0 + k + q;
      if (j >= 0 && j < n) acc = fmaf(wk[q], __ldg(in + idx + (long long)(j - pos) * stride), acc);
    }
  }
  out[idx] = accumulate ? out[idx] + acc : acc;
}

lfm_status launch_shear(const ShearPass& sp, int dir, const float* in, float* out, int nx, int ny, int nz,
                        int accumulate, void* stream, std::string& err) {
  long long nvox = (long long)nx * ny * nz;
  dim3 grid((unsigned)((nvox + 255) / 256));
  cudaStream_t s = (cudaStream_t)stream;
  if (sp.taps == 4)
    shear_kernel<4><<<grid, 256, 0, s>>>(in, out, sp.d_mlo[dir], sp.d_w[dir], sp.axis, nx, ny, nz, accumulate);
  else if (sp.taps == 8)
    shear_kernel<8><<<grid, 256, 0, s>>>(in, out, sp.d_mlo[dir], sp.d_w[dir], sp.axis, nx, ny, nz, accumulate);
  else
    shear_kernel<16><<<grid, 256, 0, s>>>(in, out, sp.d_mlo[dir], sp.d_w[dir], sp.axis, nx, ny, nz, accumulate);
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

__global__ void fill_kernel(float* __restrict__ out, long long n, float v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = v;
}

__global__ void mul_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                           long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}

constexpr int RED_BLOCKS = 592;  // 4 x 148 SMs
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

// stats: [sum w y Ax, sum w y y, sum w Ax Ax]
__global__ void __launch_bounds__(RED_THREADS) stats_partial_kernel(const float* __restrict__ Ax,
                                                                    const float* __restrict__ y,
                                                                    const float* __restrict__ w, long long n,
                                                                    double* part) {
  double v[3] = {0, 0, 0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double a = Ax[i], yy = y[i], ww = w[i];
    v[0] += ww * yy * a;
    v[1] += ww * yy * yy;
    v[2] += ww * a * a;
  }
  block_sum_store<3>(v, part);
}

__global__ void reduce_final_kernel(const double* __restrict__ part, int nblocks, int nv, double* out, int accumulate) {
  // one thread per value, fixed order: deterministic
  int q = threadIdx.x;
  if (q >= nv) return;
  double s = 0;
  for (int b = 0; b < nblocks; ++b) s += part[(size_t)b * nv + q];
  out[q] = accumulate ? out[q] + s : s;
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

// r = w (Ax - gamma y); partial 1/2 sum w (Ax - gamma y)^2
__global__ void __launch_bounds__(RED_THREADS) residual_kernel(const float* __restrict__ Ax, const float* __restrict__ y,
                                                               const float* __restrict__ w,
                                                               const double* __restrict__ gamma, int cam,
                                                               float* __restrict__ r, long long n, double* part) {
  const float g = (float)gamma[cam];
  double v[1] = {0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float d = Ax[i] - g * y[i];
    r[i] = w[i] * d;
    if (part) v[0] += 0.5 * (double)w[i] * (double)d * (double)d;
  }
  if (part) block_sum_store<1>(v, part);
}

// grad += beta * sum_{l in N_j, in grid} (x_j - x_l) + nu;  partial [nu*x_j + (beta/4) sum_l (x_j-x_l)^2]
__global__ void __launch_bounds__(RED_THREADS) reg26_kernel(const float* __restrict__ x, float* __restrict__ grad,
                                                            int nx, int ny, int nz, float beta, float nu,
                                                            double* part) {
  long long n = (long long)nx * ny * nz;
  double v[1] = {0};
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int ix = (int)(i % nx);
    long long r = i / nx;
    int iy = (int)(r % ny), iz = (int)(r / ny);
    float xj = x[i];
    float g = 0.f;
    double rs = 0;
    for (int dz = -1; dz <= 1; ++dz) {
      int zz = iz + dz;
      if (zz < 0 || zz >= nz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        int yy = iy + dy;
        if (yy < 0 || yy >= ny) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          int xx = ix + dx;
          if (xx < 0 || xx >= nx || (dx == 0 && dy == 0 && dz == 0)) continue;
          float d = xj - x[((long long)zz * ny + yy) * nx + xx];
          g += d;
          rs += (double)d * (double)d;
        }
      }
    }
    grad[i] += beta * g + nu;
    if (part) v[0] += (double)nu * xj + 0.25 * (double)beta * rs;
  }
  if (part) block_sum_store<1>(v, part);
}

__global__ void fista_kernel(float* __restrict__ x, float* __restrict__ z, const float* __restrict__ grad,
                             const float* __restrict__ d, long long n, float tau) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float xn = fmaxf(0.f, z[i] - grad[i] / d[i]);
    z[i] = xn + tau * (xn - x[i]);
    x[i] = xn;
  }
}

__global__ void majoriser_finish_kernel(float* __restrict__ d, long long n, float add) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = fmaxf(d[i] + add, 1e-12f);
}

static unsigned ew_grid(long long n) { return (unsigned)std::min<long long>((n + 255) / 256, 148 * 16); }

lfm_status k_copy_scale(const float* in, float* out, long long n, float scale, int acc, void* s, std::string& err) {
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
lfm_status k_stats(const float* Ax, const float* y, const float* w, long long n, double* part, double* out, void* s,
                   std::string& err) {
  stats_partial_kernel<<<RED_BLOCKS, RED_THREADS, 0, (cudaStream_t)s>>>(Ax, y, w, n, part);
  reduce_final_kernel<<<1, 32, 0, (cudaStream_t)s>>>(part, RED_BLOCKS, 3, out, 0);
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
  residual_kernel<<<RED_BLOCKS, RED_THREADS, 0, (cudaStream_t)s>>>(Ax, y, w, gamma, cam, r, n, cost ? part : nullptr);
  ++g_launches;
  if (cost) {
    reduce_final_kernel<<<1, 32, 0, (cudaStream_t)s>>>(part, RED_BLOCKS, 1, cost, cost_acc);
    ++g_launches;
  }
  return cuda_check(cudaGetLastError(), "residual", err);
}
lfm_status k_reg26(const float* x, float* grad, int nx, int ny, int nz, float beta, float nu, double* part,
                   double* cost, void* s, std::string& err) {
  reg26_kernel<<<RED_BLOCKS, RED_THREADS, 0, (cudaStream_t)s>>>(x, grad, nx, ny, nz, beta, nu, cost ? part : nullptr);
  ++g_launches;
  if (cost) {
    reduce_final_kernel<<<1, 32, 0, (cudaStream_t)s>>>(part, RED_BLOCKS, 1, cost, 0);
    ++g_launches;
  }
  return cuda_check(cudaGetLastError(), "reg26", err);
}
lfm_status k_fista(float* x, float* z, const float* grad, const float* d, long long n, float tau, void* s,
                   std::string& err) {
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
