// band_v: the s passes of the two-pass collapsed path on the tcgen05 tensor cores (kind::tf32, 3xTF32),
// the data as the MMA's A operand (M = 128 voxel rows vt of one slice), a banded s composite as B:
//
//   forward (DIR 0)  U[vt][n][s]   = sum_vx x[n][vt][vx] Cf_n[s][vx]        N = 256 detector columns s, K = vx
//   adjoint (DIR 1)  x[n][vt][vx] (+)= scale sum_s Z[vt][n][s] Ca_n[vx][s]   N = 16 voxel columns vx,  K = s
//
// One work item = (slice n, row tile of 128 vt, N-tile); its K range (the union of the N-tile's supports) is
// covered by blocks of BK = 16 or 32 (upload_camera, kernels.cu) with per block the N x BK weights pre-split into
// tf32 hi/lo images in the K-major swizzled layout (64-byte for BK 16, 128-byte for BK 32).  Per block the
// producer bulk-copies the images and loads the data tile [128 vt][BK k] with one 3D TMA (same swizzle = the
// same UMMA layout), the split warps write
// A_lo = A - trunc(A), the MMA thread issues per 8-wide k-step  D += A_hi B_lo + A_lo B_hi + A_hi B_hi
// (M128 N K8; for N <= 128 as two MMAs, A_hi [B_hi; B_lo] with N' = 2N and A_lo B_hi, the halves summed in the
// drain), and every `group` blocks the TMEM accumulator is drained into fp32 registers (the accumulator
// truncates, see band_u.cuh).  The epilogue writes through shared memory and 3D TMA stores (U: boxes of
// 32 s x 32 vt; x: 8 vx x 32 vt), or TMA reduce-adds when accumulating.  Warp roles as in band_u.
#pragma once
#include <cuda.h>

#include <cuda_fp16.h>

#include "tc_sm100.h"

namespace lfm {

struct VArgs {
  const float* B;          // weight images: block b at B + b * 32 * N floats (hi N x 16, then lo N x 16)
  const uint16_t* H;       // IN16: fp16 weight images (2^wexp w split into hi + lo), block b at H + 2 b BK N
  const int32_t* blk_off;  // per item key (n * n_nt + nt): blocks [off, off+1)
  const int32_t* blk_k0;   // per block: first k (vx forward, s adjoint)
  int nz, n_mt, n_nt;      // table N-tiles per slice; items = nz * n_mt * nt_cnt, (n, mt, nt0 + j)
  int nt0, nt_cnt;         // the N-tiles this launch covers (column windows of the forward)
  int k_lo, k_hi;          // K window (adjoint column windows): blocks outside [k_lo, k_hi) are skipped and the data
                           // map starts at k_lo (TMA coordinate k - k_lo; columns outside read as zeros)
  int group;               // blocks per TMEM accumulator before it is drained
  float scale;
  int accumulate;
  const float* amax;       // LFM_AMAX_SLOTS partial maxima of the source of the data (x^r forward, y adjoint)
  float amax_scale;        // OUT16 (forward): bound on the s composite's row sums -- U is written as fp16 hi + lo of
                           // 2^e U, e = u_data_exp(amax, amax_scale) (tc_sm100.h)
  float in_scale;          // IN16: the data arrives as fp16 hi + lo of 2^e data, e = u_data_exp(amax, in_scale)
  const float* rinv;       // IN16 forward: per data row (n ny + vt) scales instead: the row was split as 2^e_row x,
  int ny;                  // rinv[row] = 2^-e_row (split16_rows_kernel)
};


// live blocks [lb0, lb1) of item key: blocks are stored with ascending k0, so the ones meeting the K window are
// one contiguous run
template <bool KWIN>
__device__ __forceinline__ void v_live(const VArgs& a, int key, int BK, int& lb0, int& lb1) {
  const int b0 = __ldg(a.blk_off + key), b1 = __ldg(a.blk_off + key + 1);
  if (!KWIN) {  // no K window: every block
    lb0 = b0;
    lb1 = b1;
    return;
  }
  lb0 = b0;
  while (lb0 < b1 && __ldg(a.blk_k0 + lb0) + BK <= a.k_lo) ++lb0;
  lb1 = lb0;
  while (lb1 < b1 && __ldg(a.blk_k0 + lb1) < a.k_hi) ++lb1;
}

constexpr int V_THREADS = 384;

// H: 2xFP16 operands (data and weights pre-split into fp16 hi / lo); O16: fp16 hi / lo output (the forward's U),
// stored in boxes of 64 columns (128-byte rows, whole cache lines) from one staging buffer per warp
template <int N, int BK, bool H = false, bool O16 = false>
struct VCfg {
  static constexpr bool W64 = O16 && H;               // 64-column fp16 store boxes (2xFP16 in and out)
  static constexpr int ES = H ? 2 : 4;                // operand element bytes
  static constexpr int A_BYTES = 128 * BK * ES;       // data tile [128][BK] (hi, or lo)
  static constexpr int B_BYTES = N * BK * ES;         // one weight image [N][BK]
  static constexpr int EC0 = N >= 256 ? 128 : N / 2;
  // staging per store: 32 rows x 32 fp32 columns, or (H: fp16 hi + lo output) 32 rows x 32 fp16 columns, twice
  static constexpr int OUT0 = W64 ? 2 * 32 * 64 * 2 : 32 * (EC0 >= 32 ? 32 : EC0) * 4;
  // staging buffers per epilogue warp: 2 (store i+1 overlaps store i) when the ring keeps >= 2 stages, else 1
  // (W64: one 8 KB buffer; two with a 2-stage ring measured the same, 39.9 vs 40.0 us)
  static constexpr int NOB = W64 ? 1 : (230912 - 16 * OUT0) / (2 * A_BYTES + 2 * B_BYTES) >= 2 ? 2 : 1;
  static constexpr int RING = 230912 - 8 * NOB * OUT0;  // 227 KB minus alignment slack and barriers
  static constexpr int STAGES = RING / (2 * A_BYTES + 2 * B_BYTES) > 10 ? 10 : RING / (2 * A_BYTES + 2 * B_BYTES);
  static constexpr int SUB = BK * ES <= 128 ? BK : 128 / ES;  // sub-block width: one swizzle atom row (<= 128 B)
  static constexpr int KS = BK / SUB;
  static constexpr int SUBA = 128 * SUB * ES;         // bytes of one data sub-tile [128][SUB]
  static constexpr int SUBB = N * SUB * ES;           // bytes of one weight sub-image [N][SUB]
  static constexpr int LAYOUT = SUB * ES == 128 ? 2 : 4;  // UMMA K-major 128-byte or 64-byte swizzle
  static constexpr int SBO = 8 * SUB * ES;            // 8-row core-matrix group stride
  static constexpr int KSTEP = 32 / ES;               // K per MMA (8 tf32, 16 fp16): 32 bytes of a row
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // A | A_lo | B_hi | B_lo
  static constexpr int EC = N >= 256 ? 128 : N / 2;   // epilogue columns per warp (8 warps: 4 quarters x 2 halves)
  static constexpr int OC = W64 ? 64 : EC >= 32 ? 32 : EC;  // columns per TMA store box
  static constexpr int OUT = OUT0;                    // staging per warp and buffer
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + 8 * NOB * OUT + 1024 + 512;
  static_assert(STAGES >= 2, "band_v: stage too large");
#ifndef BAND_V_NO_MERGE
  // merged products (N <= 128, one sub-block per stage): the hi and lo weight images are consecutive K-major
  // row groups, so [B_hi; B_lo] is one N' = 2N operand and A_hi B_hi, A_hi B_lo come from one MMA (A_hi read once)
  static constexpr bool MERGE = N <= 128 && KS == 1;
#else
  static constexpr bool MERGE = false;
#endif
  static constexpr int ACC = MERGE ? 2 * N : N;      // TMEM columns per accumulator
  static constexpr int TCOLS = 2 * ACC <= 32 ? 32 : 2 * ACC <= 64 ? 64 : 2 * ACC <= 128 ? 128 : 2 * ACC <= 256 ? 256 : 512;
};

template <int N, int DIR, int BK, bool KWIN = false, bool OUT16 = false, bool IN16 = false>
__global__ void __launch_bounds__(V_THREADS, 1) band_v_kernel(const __grid_constant__ CUtensorMap a_map,
                                                              const __grid_constant__ CUtensorMap out_map,
                                                              const __grid_constant__ CUtensorMap lo_map,
                                                              const __grid_constant__ CUtensorMap a_lo_map, VArgs a) {
  using namespace tc;
  using C = VCfg<N, BK, IN16, OUT16>;
  static_assert(!OUT16 || (DIR == 0 && N == 256), "fp16 output: forward, 256-column tiles");
  extern __shared__ uint8_t v_smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)v_smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sout = sm + C::STAGES * C::STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sout + 8 * C::NOB * C::OUT);
  uint64_t* full = bars;
  uint64_t* conv = bars + C::STAGES;
  uint64_t* empty = bars + 2 * C::STAGES;
  uint64_t* tfull = bars + 3 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 64);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_barrier_init();
    prefetch_tma_desc(&a_map);
    prefetch_tma_desc(&out_map);
  }
  if (warp == 1) tmem_alloc<C::TCOLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_items = a.nz * a.n_mt * a.nt_cnt;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int nt = a.nt0 + it % a.nt_cnt, mt = (it / a.nt_cnt) % a.n_mt, n = it / (a.nt_cnt * a.n_mt);
        const int key = n * a.n_nt + nt;
        int b0, b1;
        v_live<KWIN>(a, key, BK, b0, b1);
        for (int b = b0; b < b1; ++b) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = sm + s * C::STAGE;
          mbar_arrive_expect_tx(&full[s], (IN16 ? 2 : 1) * C::A_BYTES + 2 * C::B_BYTES);
          if constexpr (IN16) bulk_g2s(st + 2 * C::A_BYTES, a.H + (size_t)b * 2 * BK * N, 2 * C::B_BYTES, &full[s]);
          else bulk_g2s(st + 2 * C::A_BYTES, a.B + (size_t)b * 2 * BK * N, 2 * C::B_BYTES, &full[s]);
          const int k = __ldg(a.blk_k0 + b) - (KWIN ? a.k_lo : 0);
#pragma unroll
          for (int j = 0; j < C::KS; ++j) {
            if (DIR == 0) tma_load_3d(st + j * C::SUBA, &a_map, k + j * C::SUB, mt * 128, n, &full[s]);   // (vx, vt, n)
            else tma_load_3d(st + j * C::SUBA, &a_map, k + j * C::SUB, n, mt * 128, &full[s]);            // (s, n, vt)
            if constexpr (IN16) {  // the pre-split lo tile beside it
              if (DIR == 0) tma_load_3d(st + C::A_BYTES + j * C::SUBA, &a_lo_map, k + j * C::SUB, mt * 128, n, &full[s]);
              else tma_load_3d(st + C::A_BYTES + j * C::SUBA, &a_lo_map, k + j * C::SUB, n, mt * 128, &full[s]);
            }
          }
          if (++s == C::STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = IN16 ? idesc_f16(128, N, 0, 0) : idesc_tf32(128, N, 0, 0);
      constexpr uint32_t IDESC2 = IN16 ? idesc_f16(128, C::MERGE ? 2 * N : N, 0, 0) : idesc_tf32(128, C::MERGE ? 2 * N : N, 0, 0);
      const uint64_t d0 = smem_desc(smem_u32(sm), 16, C::SBO, C::LAYOUT);  // all operands K-major, same swizzle
      int s = 0;
      uint32_t ph = 0;
      int buf = 0;
      uint32_t tph = 0;  // phase bit of accumulator buffer b at bit b
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int nt = a.nt0 + it % a.nt_cnt, n = it / (a.nt_cnt * a.n_mt);
        const int key = n * a.n_nt + nt;
        int b0, b1;
        v_live<KWIN>(a, key, BK, b0, b1);
        for (int g0 = b0; g0 < b1; g0 += a.group) {
          mbar_wait(&tempty[buf], ((tph >> buf) & 1u) ^ 1u);
          tph ^= 1u << buf;
          tc_fence_after();
          const uint32_t d = tmem + buf * C::ACC;
          const int g1 = min(b1, g0 + a.group);
          for (int j = g0; j < g1; ++j) {
            mbar_wait(IN16 ? &full[s] : &conv[s], ph);  // 2xFP16: the data arrives split
            tc_fence_after();
            const uint64_t so = (uint64_t)((s * C::STAGE) >> 4);  // stage offset in the descriptors' address field
#pragma unroll
            for (int kq = 0; kq < BK / C::KSTEP; ++kq) {
              const int sj = kq / (C::SUB / C::KSTEP), kk = kq % (C::SUB / C::KSTEP);
              const uint64_t ao = (uint64_t)((sj * C::SUBA + 32 * kk) >> 4), bo = (uint64_t)((sj * C::SUBB + 32 * kk) >> 4);
              const uint64_t ahi = d0 + so + ao;
              const uint64_t alo = d0 + so + (C::A_BYTES >> 4) + ao;
              const uint64_t bhi = d0 + so + ((2 * C::A_BYTES) >> 4) + bo;
              const uint64_t blo = d0 + so + ((2 * C::A_BYTES + C::B_BYTES) >> 4) + bo;
              if constexpr (IN16) {
                if constexpr (C::MERGE) {
                  mma_bf16_ss(d, ahi, bhi, IDESC2, (j != g0 || kq != 0) ? 1u : 0u);
                  mma_bf16_ss(d, alo, bhi, IDESC, 1u);
                } else {
                  mma_bf16_ss(d, ahi, blo, IDESC, (j != g0 || kq != 0) ? 1u : 0u);
                  mma_bf16_ss(d, alo, bhi, IDESC, 1u);
                  mma_bf16_ss(d, ahi, bhi, IDESC, 1u);
                }
              } else if constexpr (C::MERGE) {
                // D[:, 0:N] += A_hi B_hi, D[:, N:2N] += A_hi B_lo (one MMA), then D[:, 0:N] += A_lo B_hi
                mma_tf32_ss(d, ahi, bhi, IDESC2, (j != g0 || kq != 0) ? 1u : 0u);
                mma_tf32_ss(d, alo, bhi, IDESC, 1u);
              } else {
                mma_tf32_ss(d, ahi, blo, IDESC, (j != g0 || kq != 0) ? 1u : 0u);
                mma_tf32_ss(d, alo, bhi, IDESC, 1u);
                mma_tf32_ss(d, ahi, bhi, IDESC, 1u);
              }
            }
            tc_commit(&empty[s]);
            if (++s == C::STAGES) { s = 0; ph ^= 1; }
          }
          tc_commit(&tfull[buf]);
          buf ^= 1;
        }
      }
    }
  } else if (warp < 4) {
    if constexpr (!IN16) {  // (2xFP16: nothing to split)
    // lo split of the data tile: 128 x BK floats, 64 threads
    const int t = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int nt = a.nt0 + it % a.nt_cnt, n = it / (a.nt_cnt * a.n_mt);
      const int key = n * a.n_nt + nt;
      int lb0, lb1;
      v_live<KWIN>(a, key, BK, lb0, lb1);
      const int nb = lb1 - lb0;
      for (int b = 0; b < nb; ++b) {
        mbar_wait(&full[s], ph);
        const float4* src = reinterpret_cast<const float4*>(sm + s * C::STAGE);
        float4* lo = reinterpret_cast<float4*>(sm + s * C::STAGE + C::A_BYTES);
        constexpr int NB = BK / 2, BAT = NB < 8 ? NB : 8;  // float4 per thread, loads issued together
#pragma unroll
        for (int h = 0; h < NB / BAT; ++h) {
          float4 u[BAT];
#pragma unroll
          for (int i = 0; i < BAT; ++i) u[i] = src[t + 64 * (BAT * h + i)];
#pragma unroll
          for (int i = 0; i < BAT; ++i) {
            float4 l;
            l.x = u[i].x - __uint_as_float(__float_as_uint(u[i].x) & 0xffffe000u);
            l.y = u[i].y - __uint_as_float(__float_as_uint(u[i].y) & 0xffffe000u);
            l.z = u[i].z - __uint_as_float(__float_as_uint(u[i].z) & 0xffffe000u);
            l.w = u[i].w - __uint_as_float(__float_as_uint(u[i].w) & 0xffffe000u);
            lo[t + 64 * (BAT * h + i)] = l;
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&conv[s]);
        if (++s == C::STAGES) { s = 0; ph ^= 1; }
      }
    }
    }
  } else {
    // drain + epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (voxel rows), columns [h EC, (h+1) EC)
    constexpr int EC = C::EC, OC = C::OC;
    const int q = warp & 3, h = (warp - 4) >> 2;
    uint8_t* stg0 = sout + (warp - 4) * C::NOB * C::OUT;
    int ob = 0;  // staging buffer of the next store
    int buf = 0;
    uint32_t tph = 0;  // phase bit of accumulator buffer b at bit b
    float sig = 1.f;  // OUT16: the data scale 2^e of the 2xFP16 t pass that reads U
    if constexpr (OUT16) sig = pow2f(u_data_exp(a.amax, LFM_AMAX_SLOTS, a.amax_scale));
    float in_inv = 1.f;  // IN16: 2^-e of the data's scale (the weights' 2^-wexp is folded into a.scale)
    if constexpr (IN16) in_inv = pow2f(-u_data_exp(a.amax, LFM_AMAX_SLOTS, a.in_scale));
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int nt = a.nt0 + it % a.nt_cnt, mt = (it / a.nt_cnt) % a.n_mt, n = it / (a.nt_cnt * a.n_mt);
      const int key = n * a.n_nt + nt;
      int b0, b1;
      v_live<KWIN>(a, key, BK, b0, b1);
      float acc[EC];
#pragma unroll
      for (int c = 0; c < EC; ++c) acc[c] = 0.f;
      // IN16 forward: this lane's voxel-row scale 2^-e_row, loaded before the MMAs are waited for
      float f_row = in_inv;
      if constexpr (IN16)
        if (a.rinv) {
          const int vt = mt * 128 + 32 * q + lane;
          f_row = vt < a.ny ? __ldg(a.rinv + (size_t)n * a.ny + vt) : 1.f;
        }
      for (int g0 = b0; g0 < b1; g0 += a.group) {
        mbar_wait(&tfull[buf], (tph >> buf) & 1u);
        tph ^= 1u << buf;
        tc_fence_after();
        const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + buf * C::ACC + h * EC;
#pragma unroll
        for (int part = 0; part < (C::MERGE ? 2 : 1); ++part) {  // merged: the A_hi B_lo half at column + N
          if constexpr (EC >= 16) {
#pragma unroll
            for (int c = 0; c < EC; c += 16) {
              float v[16];
              tmem_ld16(base + part * N + c, v);
#pragma unroll
              for (int i = 0; i < 16; ++i) acc[c + i] += v[i];
            }
          } else {
            float v[EC];
            tmem_ld_n<EC>(base + part * N, v);
#pragma unroll
            for (int i = 0; i < EC; ++i) acc[i] += v[i];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        buf ^= 1;
      }
      // one multiplier per value: the data scale (a power of two: 2^-e_row or 2^-e) times scale, times the U scale
      // 2^e (OUT16) -- bit-identical to applying them one after another (powers of two commute with the rounding)
      const float mul = (IN16 ? f_row : 1.f) * a.scale * (OUT16 ? sig : 1.f);
      const int vt0 = mt * 128 + 32 * q, c0 = nt * N + h * EC;
#pragma unroll
      for (int c = 0; c < EC; c += OC) {
        uint8_t* stg = stg0 + ob * C::OUT;
        if (lane == 0) bulk_wait_read<C::NOB - 1>();  // the store that last used this buffer has read it
        __syncwarp();
        if constexpr (OUT16) {  // fp16 hi / lo of 2^e U: two 32 x OC tiles, 2 OC-byte rows, 2 OC-byte swizzle
          constexpr int RB = 2 * OC, HB = 32 * RB;  // row bytes, bytes of one half (hi or lo)
#pragma unroll
          for (int jj = 0; jj < OC / 8; ++jj) {
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float x0 = mul * acc[c + 8 * jj + 2 * i], x1 = mul * acc[c + 8 * jj + 2 * i + 1];
              const __half2 hh = __floats2half2_rn(x0, x1);
              const float2 hf = __half22float2(hh);
              const __half2 ll = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
              hw[i] = *reinterpret_cast<const uint32_t*>(&hh);
              lw[i] = *reinterpret_cast<const uint32_t*>(&ll);
            }
            const int o = RB == 128 ? lane * 128 + ((jj ^ (lane & 7)) << 4) : lane * 64 + ((jj ^ ((lane >> 1) & 3)) << 4);
            *reinterpret_cast<uint4*>(stg + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(stg + HB + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
        } else if constexpr (OC == 32) {  // 128-byte rows, 128-byte swizzle
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const float4 v = make_float4(mul * acc[c + 4 * jj], mul * acc[c + 4 * jj + 1], mul * acc[c + 4 * jj + 2],
                                         mul * acc[c + 4 * jj + 3]);
            *reinterpret_cast<float4*>(stg + lane * 128 + ((jj ^ (lane & 7)) << 4)) = v;
          }
        } else {  // OC-float rows, no swizzle
#pragma unroll
          for (int jj = 0; jj < OC; jj += 4) {
            const float4 v = make_float4(mul * acc[c + jj], mul * acc[c + jj + 1], mul * acc[c + jj + 2],
                                         mul * acc[c + jj + 3]);
            *reinterpret_cast<float4*>(stg + lane * OC * 4 + jj * 4) = v;
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (OUT16) {  // U hi / lo maps (s, n, vt), fp16
            tma_store_3d(&out_map, c0 + c, n, vt0, stg);
            tma_store_3d(&lo_map, c0 + c, n, vt0, stg + 32 * 2 * OC);
          } else if (DIR == 0) {  // U map (s, n, vt)
            if (a.accumulate) tma_add_3d(&out_map, c0 + c, n, vt0, stg);
            else tma_store_3d(&out_map, c0 + c, n, vt0, stg);
          } else {  // x map (vx, vt, n)
            if (a.accumulate) tma_add_3d(&out_map, c0 + c, vt0, n, stg);
            else tma_store_3d(&out_map, c0 + c, vt0, n, stg);
          }
          bulk_commit();
        }
        if (++ob == C::NOB) ob = 0;
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::TCOLS>(tmem);
}

}  // namespace lfm
