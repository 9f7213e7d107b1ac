// Direct s passes of the two-pass collapsed path, HBM-bound, no transposes:
//
//   forward  U[vt][n][s]  = sum_e Cf_n[s][e] x_n[vt][j_e]             (slice n of the rotated volume -> the
//                                                                       interleaved intermediate the t pass reads)
//   adjoint  x_n[vt][vx] (+)= scale sum_e Ca_n[vx][e] Z[vt][n][s_e]     (the t pass's output -> slice n)
//
// Cf_n / Ca_n are the per-slice s composites (plan families cf[0] / ca[0]) in their ELL form
// ([table][entry][row], exact non-zeros in increasing source order, rows padded to a multiple of 4).
//
// spass_fwd_kernel: CTA = (256 detector columns s, slice n, 32 voxel rows).  The 32 rows of x_n are staged
//   transposed in shared memory (xsT[vx][vt], lanes over vt on the store side: conflict-free), so each of a
//   thread's entries (j, w) feeds 32 outputs from 8 LDS.128; consecutive threads on consecutive s store
//   128-byte rows.  The 128 MiB write of U is the roofline.
// spass_adj_kernel: CTA = (16 voxel columns vx, slice n), looping over the 4 groups of 32 voxel rows and over
//   128-column chunks of the 16 columns' source footprint: the chunk of Z is staged with an odd row stride, a
//   lane owns a voxel row (conflict-free), the taps of the CTA's 16 columns sit in shared memory (warp-uniform
//   broadcasts); results leave through shared memory as 64-byte row segments.
#pragma once

namespace lfm {

constexpr int SPF_VTG = 32;   // voxel rows per forward CTA
constexpr int SPA_VX = 16;    // voxel columns per adjoint CTA
constexpr int SPA_VT = 32;    // voxel rows per adjoint group (one per lane)
constexpr int SPA_CH = 128;   // source columns per staged adjoint chunk

__global__ void __launch_bounds__(256) spass_fwd_kernel(const float* __restrict__ x, float* __restrict__ U,
                                                        const int32_t* __restrict__ cnt, const int32_t* __restrict__ idx,
                                                        const float* __restrict__ w, int nx, int ny, int nz, int nd,
                                                        int ell, int pitch) {
  extern __shared__ float4 xs4[];  // xsT[vx][32 vt] as float4 groups of 4 voxel rows
  float* xsT = reinterpret_cast<float*>(xs4);
  const int n = blockIdx.y, vt0 = blockIdx.z * SPF_VTG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* xn = x + ((size_t)n * ny + vt0) * nx;
  const bool row_in = vt0 + lane < ny;
  // lane = voxel row, 4 consecutive vx per load; warps split the vx range
  for (int j0 = 4 * warp; j0 < nx; j0 += 32) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row_in) {
      const float* p = xn + (size_t)lane * nx + j0;
      if (j0 + 4 <= nx && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) v = __ldg(reinterpret_cast<const float4*>(p));
      else {
        v.x = __ldg(p);
        if (j0 + 1 < nx) v.y = __ldg(p + 1);
        if (j0 + 2 < nx) v.z = __ldg(p + 2);
        if (j0 + 3 < nx) v.w = __ldg(p + 3);
      }
    }
    xsT[(j0 + 0) * SPF_VTG + lane] = v.x;
    if (j0 + 1 < nx) xsT[(j0 + 1) * SPF_VTG + lane] = v.y;
    if (j0 + 2 < nx) xsT[(j0 + 2) * SPF_VTG + lane] = v.z;
    if (j0 + 3 < nx) xsT[(j0 + 3) * SPF_VTG + lane] = v.w;
  }
  __syncthreads();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nd) return;
  const int32_t* ip = idx + (size_t)n * ell * pitch + s;
  const float* wp = w + (size_t)n * ell * pitch + s;
  const int c = __ldg(cnt + (size_t)n * pitch + s);
  float acc[SPF_VTG];
#pragma unroll
  for (int r = 0; r < SPF_VTG; ++r) acc[r] = 0.f;
  // entries in groups of 4 (ELL rows are padded to a multiple of 4 with zero weights): the 8 loads of a group
  // are independent, so one memory latency per group instead of one per entry
  for (int e = 0; e < c; e += 4) {
    int j[4];
    float wv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      j[k] = __ldg(ip + (size_t)(e + k) * pitch);
      wv[k] = __ldg(wp + (size_t)(e + k) * pitch);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4* col = xs4 + j[k] * (SPF_VTG / 4);
#pragma unroll
      for (int g = 0; g < SPF_VTG / 4; ++g) {
        const float4 v = col[g];
        acc[4 * g] = fmaf(wv[k], v.x, acc[4 * g]);
        acc[4 * g + 1] = fmaf(wv[k], v.y, acc[4 * g + 1]);
        acc[4 * g + 2] = fmaf(wv[k], v.z, acc[4 * g + 2]);
        acc[4 * g + 3] = fmaf(wv[k], v.w, acc[4 * g + 3]);
      }
    }
  }
  float* u = U + ((size_t)vt0 * nz + n) * nd + s;
  const size_t rstep = (size_t)nz * nd;
  const int nr = min(SPF_VTG, ny - vt0);
  if (nr == SPF_VTG) {
#pragma unroll
    for (int r = 0; r < SPF_VTG; ++r, u += rstep) *u = acc[r];
  } else {
#pragma unroll
    for (int r = 0; r < SPF_VTG; ++r, u += rstep)
      if (r < nr) *u = acc[r];
  }
}

// fp[n * n_tiles + tile] = {first s, width} of the union of the tile's rows' non-zero columns (plan-time, host);
// taps per row <= tmax (shared-memory tap table [SPA_VX][tmax]).
__global__ void __launch_bounds__(256) spass_adj_kernel(const float* __restrict__ Z, float* __restrict__ out,
                                                        const int32_t* __restrict__ cnt, const int32_t* __restrict__ idx,
                                                        const float* __restrict__ w, const int2* __restrict__ fp,
                                                        int nx, int ny, int nz, int nd, int ell, int pitch, int tmax,
                                                        float scale, int accumulate) {
  extern __shared__ float sm[];
  float* zs = sm;                                   // [SPA_VT][SPA_CH + 1]
  float* res = zs + SPA_VT * (SPA_CH + 1);          // [SPA_VT][SPA_VX + 1]
  float* tw = res + SPA_VT * (SPA_VX + 1);          // [SPA_VX][tmax] weights
  int* tj = reinterpret_cast<int*>(tw + SPA_VX * tmax);  // [SPA_VX][tmax] source columns
  __shared__ int tc[SPA_VX];
  const int tile = blockIdx.x, n = blockIdx.y;
  const int n_tiles = gridDim.x;
  const int2 f = __ldg(fp + (size_t)n * n_tiles + tile);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // taps of the 16 columns
  for (int i = threadIdx.x; i < SPA_VX * tmax; i += blockDim.x) {
    const int lx = i / tmax, e = i - lx * tmax, vx = tile * SPA_VX + lx;
    const int c = vx < nx ? __ldg(cnt + (size_t)n * pitch + vx) : 0;
    if (e == 0) tc[lx] = c;
    const size_t o = (size_t)n * ell * pitch + (size_t)e * pitch + vx;
    tj[i] = e < c ? __ldg(idx + o) : 0;
    tw[i] = e < c ? __ldg(w + o) : 0.f;
  }
  __syncthreads();
  for (int vt0 = 0; vt0 < ny; vt0 += SPA_VT) {
    float acc[SPA_VX / 8] = {0.f, 0.f};
    int ep[SPA_VX / 8] = {0, 0};
    for (int c0 = f.x; c0 < f.x + f.y; c0 += SPA_CH) {
      const int cw = min(SPA_CH, f.x + f.y - c0);
      // stage Z[vt0 + r][n][c0 .. c0 + cw) : one warp per row, coalesced
      for (int r = warp; r < SPA_VT; r += 8) {
        const bool in = vt0 + r < ny;
        const float* zr = Z + ((size_t)(vt0 + r) * nz + n) * nd + c0;
        for (int i = lane; i < cw; i += 32) zs[r * (SPA_CH + 1) + i] = in ? __ldg(zr + i) : 0.f;
      }
      __syncthreads();
      const float* zrow = zs + lane * (SPA_CH + 1) - c0;
#pragma unroll
      for (int q = 0; q < SPA_VX / 8; ++q) {
        const int lx = warp * (SPA_VX / 8) + q;
        const int c = tc[lx];
        const int* jj = tj + lx * tmax;
        const float* ww = tw + lx * tmax;
        int e = ep[q];
        float a = acc[q];
        while (e < c && jj[e] < c0 + cw) {
          a = fmaf(ww[e], zrow[jj[e]], a);
          ++e;
        }
        ep[q] = e;
        acc[q] = a;
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < SPA_VX / 8; ++q) res[lane * (SPA_VX + 1) + warp * (SPA_VX / 8) + q] = scale * acc[q];
    __syncthreads();
    for (int i = threadIdx.x; i < SPA_VT * SPA_VX; i += blockDim.x) {
      const int r = i / SPA_VX, cx = i % SPA_VX;
      const int vt = vt0 + r, vx = tile * SPA_VX + cx;
      if (vt < ny && vx < nx) {
        float* o = out + ((size_t)n * ny + vt) * nx + vx;
        const float v = res[r * (SPA_VX + 1) + cx];
        *o = accumulate ? *o + v : v;
      }
    }
    __syncthreads();
  }
}

// spass_adj_row_kernel: one warp per Z row (vt, n) (the 8 warps of a CTA take 8 voxel rows of one slice): the
//   row is staged in warp-private shared memory with one pad word per 16 columns (the taps of consecutive vx
//   sit ~16 columns apart, so the pad makes them hit distinct banks), lane l computes vx = l, l + 32, ...
//   from the ELL taps (coalesced across lanes, L1-resident for the CTA's slice) and stores 128-byte rows.
__global__ void __launch_bounds__(256) spass_adj_row_kernel(const float* __restrict__ Z, float* __restrict__ out,
                                                            const int32_t* __restrict__ cnt, const int32_t* __restrict__ idx,
                                                            const float* __restrict__ w, int nx, int ny, int nz, int nd,
                                                            int ell, int pitch, float scale, int accumulate) {
  extern __shared__ float rs[];  // 8 warps x (nd + nd / 16 + 4)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = blockIdx.y, vt = blockIdx.x * 8 + warp;
  if (vt >= ny) return;
  const int rstride = nd + nd / 16 + 4;
  float* row = rs + warp * rstride;
  const float* zr = Z + ((size_t)vt * nz + n) * nd;
  if ((nd & 3) == 0 && ((reinterpret_cast<uintptr_t>(zr) & 15) == 0)) {
    for (int q = lane; q < nd / 4; q += 32) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(zr) + q);
      const int s0 = 4 * q, o = s0 + (s0 >> 4);
      row[o] = v.x; row[o + 1] = v.y; row[o + 2] = v.z; row[o + 3] = v.w;
    }
  } else {
    for (int s0 = lane; s0 < nd; s0 += 32) row[s0 + (s0 >> 4)] = __ldg(zr + s0);
  }
  __syncwarp();
  const size_t tb = (size_t)n * ell * pitch;
  float* o = out + ((size_t)n * ny + vt) * nx;
  for (int vx = lane; vx < nx; vx += 32) {
    const int c = __ldg(cnt + (size_t)n * pitch + vx);
    const int32_t* ip = idx + tb + vx;
    const float* wp = w + tb + vx;
    float a0 = 0.f, a1 = 0.f;
    for (int e = 0; e < c; e += 4) {
      int j[4];
      float wv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        j[k] = __ldg(ip + (size_t)(e + k) * pitch);
        wv[k] = __ldg(wp + (size_t)(e + k) * pitch);
      }
      a0 = fmaf(wv[0], row[j[0] + (j[0] >> 4)], a0);
      a1 = fmaf(wv[1], row[j[1] + (j[1] >> 4)], a1);
      a0 = fmaf(wv[2], row[j[2] + (j[2] >> 4)], a0);
      a1 = fmaf(wv[3], row[j[3] + (j[3] >> 4)], a1);
    }
    const float v = scale * (a0 + a1);
    o[vx] = accumulate ? o[vx] + v : v;
  }
}

}  // namespace lfm
