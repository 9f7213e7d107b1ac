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
#pragma once

namespace lfm {

constexpr int SPF_VTG = 32;   // voxel rows per forward CTA

__global__ void __launch_bounds__(256, 3) spass_fwd_kernel(const float* __restrict__ x, float* __restrict__ U,
                                                           const int32_t* __restrict__ cnt, const int32_t* __restrict__ idx,
                                                           const float* __restrict__ w, int nx, int ny, int nz, int nd,
                                                           int ell, int pitch) {
  extern __shared__ float4 xs4[];  // xsT[vx][32 vt] as float4 groups of 4 voxel rows
  float* xsT = reinterpret_cast<float*>(xs4);
  const int n = blockIdx.y, vt0 = blockIdx.z * SPF_VTG;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const bool s_in = s < nd;
  // this column's first entries, issued before the staging so both latencies overlap
  const int32_t* ip = idx + (size_t)n * ell * pitch + s;
  const float* wp = w + (size_t)n * ell * pitch + s;
  const int c = s_in ? __ldg(cnt + (size_t)n * pitch + s) : 0;
  int j[4];
  float wv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    j[k] = (s_in && k < ell) ? __ldg(ip + (size_t)k * pitch) : 0;
    wv[k] = (s_in && k < ell) ? __ldg(wp + (size_t)k * pitch) : 0.f;
  }
  // stage x_n rows vt0.. transposed: lane = voxel row, 4 consecutive vx per load, all loads issued first
  const float* xr = x + ((size_t)n * ny + vt0 + lane) * nx;
  const bool row_in = vt0 + lane < ny;
  constexpr int MAXJ = 8;  // nx <= 8 * 32 * ... handled in chunks of 8 float4 per lane
  for (int jb = 4 * warp; jb < nx; jb += 32 * MAXJ) {
    float4 v[MAXJ];
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) {
      const int j0 = jb + 32 * q;
      v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row_in && j0 < nx) {
        if (j0 + 4 <= nx && ((nx & 3) == 0)) v[q] = __ldg(reinterpret_cast<const float4*>(xr + j0));
        else {
          v[q].x = __ldg(xr + j0);
          if (j0 + 1 < nx) v[q].y = __ldg(xr + j0 + 1);
          if (j0 + 2 < nx) v[q].z = __ldg(xr + j0 + 2);
          if (j0 + 3 < nx) v[q].w = __ldg(xr + j0 + 3);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < MAXJ; ++q) {
      const int j0 = jb + 32 * q;
      if (j0 < nx) xsT[j0 * SPF_VTG + lane] = v[q].x;
      if (j0 + 1 < nx) xsT[(j0 + 1) * SPF_VTG + lane] = v[q].y;
      if (j0 + 2 < nx) xsT[(j0 + 2) * SPF_VTG + lane] = v[q].z;
      if (j0 + 3 < nx) xsT[(j0 + 3) * SPF_VTG + lane] = v[q].w;
    }
  }
  __syncthreads();
  if (!s_in) return;
  float acc[SPF_VTG];
#pragma unroll
  for (int r = 0; r < SPF_VTG; ++r) acc[r] = 0.f;
  for (int e = 0; e < c; e += 4) {
    // next group's loads first (independent of this group's arithmetic)
    int jn[4];
    float wn[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool more = e + 4 + k < c;
      jn[k] = more ? __ldg(ip + (size_t)(e + 4 + k) * pitch) : 0;
      wn[k] = more ? __ldg(wp + (size_t)(e + 4 + k) * pitch) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e + k < c) {
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
#pragma unroll
    for (int k = 0; k < 4; ++k) { j[k] = jn[k]; wv[k] = wn[k]; }
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

// spass_adj_kernel<VTA>: CTA = (VTA voxel rows, slice n), 128 threads.  The VTA rows Z[vt][n][:] are staged
//   in shared memory with one pad word per 16 columns (the taps of consecutive vx sit ~16 columns apart, so
//   the pad puts neighbouring lanes on distinct banks); thread = voxel column vx (lanes on consecutive vx:
//   coalesced ELL loads and 128-byte output rows), each tap (j, w) feeds VTA outputs from registers.
template <int VTA>
__global__ void __launch_bounds__(128) spass_adj_kernel(const float* __restrict__ Z, float* __restrict__ out,
                                                        const int32_t* __restrict__ cnt, const int32_t* __restrict__ idx,
                                                        const float* __restrict__ w, int nx, int ny, int nz, int nd,
                                                        int ell, int pitch, float scale, int accumulate) {
  extern __shared__ float zr[];  // [VTA][rs]
  const int n = blockIdx.y, vt0 = blockIdx.x * VTA;
  const int rs = nd + (nd >> 4) + 4;
  const int nq = nd >> 2;
  const bool vec = (nd & 3) == 0;
  for (int i = threadIdx.x; i < VTA * (vec ? nq : nd); i += blockDim.x) {
    if (vec) {
      const int r = i / nq, q = i - r * nq, s0 = 4 * q;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (vt0 + r < ny) v = __ldg(reinterpret_cast<const float4*>(Z + ((size_t)(vt0 + r) * nz + n) * nd) + q);
      float* o = zr + r * rs + s0 + (s0 >> 4);
      o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
      const int r = i / nd, s0 = i - r * nd;
      zr[r * rs + s0 + (s0 >> 4)] = vt0 + r < ny ? __ldg(Z + ((size_t)(vt0 + r) * nz + n) * nd + s0) : 0.f;
    }
  }
  __syncthreads();
  const int nr = min(VTA, ny - vt0);
  for (int vx = threadIdx.x; vx < nx; vx += blockDim.x) {
    const int c = __ldg(cnt + (size_t)n * pitch + vx);
    const int32_t* ip = idx + (size_t)n * ell * pitch + vx;
    const float* wp = w + (size_t)n * ell * pitch + vx;
    float acc[VTA];
#pragma unroll
    for (int r = 0; r < VTA; ++r) acc[r] = 0.f;
    for (int e = 0; e < c; e += 4) {
      int j[4];
      float wv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // ELL rows are padded to a multiple of 4 with zero weights
        j[k] = __ldg(ip + (size_t)(e + k) * pitch);
        wv[k] = __ldg(wp + (size_t)(e + k) * pitch);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float* zc = zr + j[k] + (j[k] >> 4);
#pragma unroll
        for (int r = 0; r < VTA; ++r) acc[r] = fmaf(wv[k], zc[r * rs], acc[r]);
      }
    }
    float* o = out + ((size_t)n * ny + vt0) * nx + vx;
#pragma unroll
    for (int r = 0; r < VTA; ++r, o += nx)
      if (r < nr) *o = accumulate ? *o + scale * acc[r] : scale * acc[r];
  }
}

}  // namespace lfm
