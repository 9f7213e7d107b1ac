// band_u: the identity-s t pass  out[r][c] = scale * sum_k C[r][k] src[k][c]  (C a banded 1D operator from
// the plan, src row-major with pitch) on the 5th-generation tensor cores (tcgen05, kind::tf32, 3xTF32).
//
// C is cut into tiles of 128 rows; the union of a tile's non-zero source rows is covered by blocks of 16
// consecutive source rows (build_umma in plan.cpp).  Per block the plan stores the 128 x 16 weights as two
// tf32 images (hi = rn(w), lo = rn(w - hi)) laid out exactly as the tensor core reads them from shared memory
// (K-major, 64-byte swizzle).  One work item = (row tile, 256 output columns); a CTA runs items persistently:
//
//   warp 0      producer: per block one bulk copy of the weight images (16 KB) and 8 TMA tiles of the source
//               (16 rows x 32 columns each, 128B/32B-atom swizzle = UMMA MN-major layout type 1)
//   warps 2-3   split: the tensor core truncates fp32 to tf32, so src = hi + lo with hi = the raw tile and
//               lo = src - trunc(src) (exact), written beside it
//   warp 1      MMA issuer: per block and 8-row k-step  D += C_lo S_hi + C_hi S_lo + C_hi S_hi  (M128 N256 K8)
//   warps 4-11  drain + epilogue: the TMEM accumulator adds by truncation (measured,
//               tools/microbench/tc_probe.cu), so a chain of MMAs drifts low by ~2^-24 per add; every `group`
//               blocks the MMA warp switches to the other of two TMEM accumulators and these warps add the
//               finished one into fp32 registers (round to nearest), then write the item's output rows.
#pragma once
#include <cuda.h>

#include <cuda_fp16.h>

#include "tc_sm100.h"

namespace lfm {

struct UArgs {
  const float* A;         // weight images: block b at A + 4096 b (hi 2048 floats, then lo 2048 floats)
  const uint16_t* H;      // 2xFP16 form (F16 instances): block b at H + 4096 b (hi 2048 halves, then lo), weights
                          // scaled by 2^wexp (the host folds 2^-wexp into `scale`)
  const float* amax;      // F16: n_amax partial maxima m_i; the source was written as fp16 hi + lo of 2^e src with
  int n_amax;             // e = u_data_exp(max m_i * amax_scale) by its producer (band_v / split16_kernel), so the
  float amax_scale;       // epilogue takes 2^-e back out
  const float* cinv;      // OUT16, optional: the source was split with a scale per column (split16_cols_kernel), the
                          // epilogue takes cinv[c] = 2^-e_c back out per output column (the t pass never mixes columns)
  float out_scale16;      // OUT16 instances: the output is written as fp16 hi + lo of 2^e' out, e' =
                          // u_data_exp(max m_i * out_scale16) (a bound on |out| over max |src| m_i: the row sums)
  const int32_t* blk_off; // per row tile: first block .. (row tiles of the table, n_tiles + 1 entries)
  const int32_t* blk_k0;  // per block: first source row (plan coordinates)
  float* out;
  long long out_pitch;
  int n_rows, n_cols;     // output rows (table rows) and columns
  int mt0, n_mt, n_nt;    // row tiles [mt0, mt0 + n_mt), column tiles of 256
  int k_shift;            // source row of TMA coordinate 0 (the row window start)
  int k_end;              // end of the source row window (k_shift + rows); blocks outside it are skipped
  int windowed;           // 1: the window is narrower than the source (row-sharded adjoint)
  int group;              // blocks per TMEM accumulator before it is drained
  float scale;
  int accumulate;
  int tile_mode;          // 0: tile = 128 consecutive rows; 1: 2 rows-of-slices (vt) x 64 slices, rows vt*nz + n
  int tm_nz;              // nz for tile_mode 1
  int nt0;                // first column tile (column windows: tiles [nt0, nt0 + n_nt))
  int ksplit;             // split-K: each (row tile, column tile) is ksplit items over consecutive thirds.. of its
                          // live blocks; chunk kc writes its partial at output row kc * kc_rows + r (kc_rows =
                          // row tiles x 128), summed in a fixed order by sum_chunks_kernel (deterministic)
  int kc_rows;
  int src3d;              // 2xFP16: the source maps are 3D (64 columns, rows, 64-column groups), one box per part
};



// blocks of row tile mt whose 16 source rows intersect the row window (all of them when not windowed)
__device__ __forceinline__ bool u_live(const UArgs& a, int b) {
  const int k = __ldg(a.blk_k0 + b);
  return k + 16 > a.k_shift && k < a.k_end;
}
__device__ __forceinline__ int u_nlive(const UArgs& a, int b0, int b1) {
  if (!a.windowed) return b1 - b0;
  int n = 0;
  for (int b = b0; b < b1; ++b) n += u_live(a, b);
  return n;
}

// item it -> (row tile, column tile, K chunk) and the chunk's live-block range [lo, hi) in producer order
struct UItem {
  int mt, nt, kc, b0, b1, lo, hi;
};
template <bool SPLIT>
__device__ __forceinline__ UItem u_item(const UArgs& a, int it) {
  UItem u;
  if constexpr (!SPLIT) {  // one item per (row tile, column tile): the whole live range
    u.mt = a.mt0 + it / a.n_nt;
    u.nt = a.nt0 + it % a.n_nt;
    u.kc = 0;
    u.b0 = __ldg(a.blk_off + u.mt);
    u.b1 = __ldg(a.blk_off + u.mt + 1);
    u.lo = 0;
    u.hi = u_nlive(a, u.b0, u.b1);
    return u;
  }
  const int per_mt = a.n_nt * a.ksplit;
  u.mt = a.mt0 + it / per_mt;
  const int rem = it % per_mt;
  u.nt = a.nt0 + rem / a.ksplit;
  u.kc = rem % a.ksplit;
  u.b0 = __ldg(a.blk_off + u.mt);
  u.b1 = __ldg(a.blk_off + u.mt + 1);
  const int nl = u_nlive(a, u.b0, u.b1);
  u.lo = (int)((long long)nl * u.kc / a.ksplit);
  u.hi = (int)((long long)nl * (u.kc + 1) / a.ksplit);
  return u;
}

constexpr int U_STAGES = 4;
constexpr int U_STAGE_BYTES = 49152;  // A hi+lo (16 KB) | src tile (16 KB) | src lo (16 KB)
// 2xFP16: A hi+lo (8 KB) | src tile fp32 (16 KB), overwritten in place by the fp16 src hi (8 KB) | src lo (8 KB)
// OUT16 (the adjoint's fp16 Z): 6 stages and 8 KB of epilogue staging per warp, so Z goes out in 64-column boxes
// (whole 128-byte lines of its fp16 rows) -- the source (the split y) is L2-resident, so fewer stages suffice
template <bool F16, bool OUT16 = false> struct UStage {
  static constexpr int STAGES = OUT16 ? 6 : F16 ? 8 : U_STAGES;
  static constexpr int OUT = OUT16 ? 8192 : 4096;  // epilogue staging per warp
  static constexpr int BYTES = F16 ? 24576 : U_STAGE_BYTES;
};
constexpr int U_THREADS = 384;

#ifndef U_SPLIT_BATCH
#define U_SPLIT_BATCH 8  // float4 loads issued together by each split thread (16 per block)
#endif
constexpr int U_STAGE_OUT = 4096;  // per epilogue warp: 32 rows x 32 columns fp32, 128-byte swizzle (TMA store)
constexpr size_t U_SMEM = (size_t)U_STAGES * U_STAGE_BYTES + 8 * U_STAGE_OUT + 1024 + 256;

template <bool SPLIT, bool F16 = false, bool OUT16 = false>
__global__ void __launch_bounds__(U_THREADS, 1) band_u_kernel(const __grid_constant__ CUtensorMap src_map,
                                                              const __grid_constant__ CUtensorMap out_map,
                                                              const __grid_constant__ CUtensorMap lo_map,
                                                              const __grid_constant__ CUtensorMap out_lo_map, UArgs a) {
  static_assert(!OUT16 || (F16 && !SPLIT), "fp16 output: 2xFP16 form, no split-K");
  using namespace tc;
  constexpr int U_STAGES = UStage<F16, OUT16>::STAGES, U_STAGE_BYTES = UStage<F16, OUT16>::BYTES;
  constexpr int U_STAGE_OUT = UStage<F16, OUT16>::OUT;
  static_assert(UStage<true>::STAGES * UStage<true>::BYTES == 4 * 49152, "same ring size");
  static_assert(UStage<F16, OUT16>::STAGES * UStage<F16, OUT16>::BYTES + 8 * U_STAGE_OUT + 1024 + 256 +
                    (OUT16 ? 4096 : 0) <= U_SMEM,
                "shared memory");
  extern __shared__ uint8_t u_smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)u_smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sout = sm + U_STAGES * U_STAGE_BYTES;  // epilogue staging, 8 x 4 KB (OUT16: 8 x 8 KB)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sout + 8 * U_STAGE_OUT);
  uint64_t* full = bars;                  // TMA landed (tx count)
  uint64_t* conv = bars + U_STAGES;       // lo split written (64 arrivals)
  uint64_t* empty = bars + 2 * U_STAGES;  // MMAs of the stage done (commit)
  uint64_t* tfull = bars + 3 * U_STAGES;  // accumulator ready (commit), 2
  uint64_t* tempty = tfull + 2;           // accumulator drained (8 warps), 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < U_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 64);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_barrier_init();
    prefetch_tma_desc(&src_map);
    prefetch_tma_desc(&out_map);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_items = a.n_mt * a.n_nt * (SPLIT ? a.ksplit : 1);

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const UItem ui = u_item<SPLIT>(a, it);
        const int mt = ui.mt, nt = ui.nt, b0 = ui.b0, b1 = ui.b1;
        const bool rev = (mt & 1) != 0;
        int li = 0;  // live-block index in producer order (split-K chunks)
        // block starts read one block ahead, so the load's latency overlaps the previous block's wait and issue
        int k_next = b0 < b1 ? __ldg(a.blk_k0 + (rev ? b1 - 1 : b0)) : 0;
        for (int j = b0; j < b1; ++j) {
          const int b = rev ? b0 + b1 - 1 - j : j;
          const int k_raw = k_next;
          if (j + 1 < b1) k_next = __ldg(a.blk_k0 + (rev ? b0 + b1 - 2 - j : j + 1));
          if (a.windowed && !(k_raw + 16 > a.k_shift && k_raw < a.k_end)) continue;  // (u_live)
          if constexpr (SPLIT) {
            const int my = li++;
            if (my < ui.lo) continue;
            if (my >= ui.hi) break;
          }
          const int k = k_raw - a.k_shift;
          uint8_t* st = sm + s * U_STAGE_BYTES;
          mbar_wait(&empty[s], ph ^ 1);
          if constexpr (F16) {  // fp16 weight images (8 KB); pre-split fp16 source hi and lo, 4 boxes of 16 rows x 64
                                // columns each with the 128-byte swizzle = the MN-major operand layout
            mbar_arrive_expect_tx(&full[s], 8192 + 16384);
            bulk_g2s(st, a.H + (size_t)b * 4096, 8192, &full[s]);
            if (a.src3d) {  // 4 column groups x 16 rows x 64 columns = the same [g][row][64] layout in one box
              tma_load_3d(st + 8192, &src_map, 0, k, nt * 4, &full[s]);
              tma_load_3d(st + 16384, &lo_map, 0, k, nt * 4, &full[s]);
            } else {
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                tma_load_2d(st + 8192 + g * 2048, &src_map, nt * 256 + g * 64, k, &full[s]);
                tma_load_2d(st + 16384 + g * 2048, &lo_map, nt * 256 + g * 64, k, &full[s]);
              }
            }
          } else {
            mbar_arrive_expect_tx(&full[s], 32768);
            bulk_g2s(st, a.A + (size_t)b * 4096, 16384, &full[s]);
#pragma unroll
            for (int g = 0; g < 8; ++g) tma_load_2d(st + 16384 + g * 2048, &src_map, nt * 256 + g * 32, k, &full[s]);
          }
          if (++s == U_STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = F16 ? idesc_f16(128, 256, 0, 1) : idesc_tf32(128, 256, 0, 1);
      // tf32: weights K-major 64-byte swizzle, source MN-major 128B/32B-atom; fp16: weights K-major 32-byte
      // swizzle, source MN-major 128-byte swizzle (atoms of 64 columns x 8 rows, 2048 bytes apart along N)
      const uint64_t dA0 = F16 ? smem_desc(smem_u32(sm), 16, 256, 6) : smem_desc(smem_u32(sm), 16, 512, 4);
      const uint64_t dB0 = F16 ? smem_desc(smem_u32(sm) + 8192, 2048, 1024, 2) : smem_desc(smem_u32(sm) + 16384, 2048, 512, 1);
      int s = 0;
      uint32_t ph = 0;
      int buf = 0;
      uint32_t tph = 0;  // phase bit of accumulator buffer b at bit b
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const UItem ui = u_item<SPLIT>(a, it);
        const int b0 = 0, b1 = ui.hi - ui.lo;  // the chunk's live blocks in producer order
        for (int g0 = b0; g0 < b1; g0 += a.group) {
          mbar_wait(&tempty[buf], ((tph >> buf) & 1u) ^ 1u);
          tph ^= 1u << buf;
          tc_fence_after();
          const uint32_t d = tmem + buf * 256;
          const int g1 = min(b1, g0 + a.group);
          for (int j = g0; j < g1; ++j) {
            mbar_wait(F16 ? &full[s] : &conv[s], ph);  // 2xFP16: the source arrives split, no split warps
            tc_fence_after();
            // descriptors = the stage-0 ones plus the start-address offset (16-byte units, low field; no carry)
            const uint64_t so = (uint64_t)((s * U_STAGE_BYTES) >> 4);
            if constexpr (F16) {  // one K = 16 step: D += C_lo S_hi + C_hi S_lo + C_hi S_hi
              const uint64_t ahi = dA0 + so, alo = dA0 + so + (4096 >> 4);
              const uint64_t bhi = dB0 + so, blo = dB0 + so + (8192 >> 4);
#ifndef BAND_U_NO_MMA
              mma_bf16_ss(d, alo, bhi, IDESC, j != g0 ? 1u : 0u);
              mma_bf16_ss(d, ahi, blo, IDESC, 1u);
              mma_bf16_ss(d, ahi, bhi, IDESC, 1u);
#endif
            } else
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const uint64_t ahi = dA0 + so + 2 * kk;
              const uint64_t alo = dA0 + so + (8192 >> 4) + 2 * kk;
              const uint64_t bhi = dB0 + so + 64 * kk;
              const uint64_t blo = dB0 + so + (16384 >> 4) + 64 * kk;
              mma_tf32_ss(d, alo, bhi, IDESC, (j != g0 || kk != 0) ? 1u : 0u);
#ifndef BAND_U_TWO_PRODUCTS
              mma_tf32_ss(d, ahi, blo, IDESC, 1u);
#endif
              mma_tf32_ss(d, ahi, bhi, IDESC, 1u);
            }
            tc_commit(&empty[s]);
            if (++s == U_STAGES) { s = 0; ph ^= 1; }
          }
          tc_commit(&tfull[buf]);
          buf ^= 1;
        }
      }
    }
  } else if (warp < 4) {
    if constexpr (!F16) {  // (2xFP16: nothing to split)
    // lo split: 16 KB source tile = 1024 float4, 64 threads x 16
    const int t = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const UItem ui = u_item<SPLIT>(a, it);
      const int nb = ui.hi - ui.lo;
      for (int b = 0; b < nb; ++b) {
        mbar_wait(&full[s], ph);
        const float4* src = reinterpret_cast<const float4*>(sm + s * U_STAGE_BYTES + 16384);
        float4* lo = reinterpret_cast<float4*>(sm + s * U_STAGE_BYTES + 32768);
#ifndef BAND_U_NO_SPLIT
        // all 16 loads first (one shared-memory latency for the block), then the 16 stores
#pragma unroll
        for (int h = 0; h < 16 / U_SPLIT_BATCH; ++h) {
          float4 u[U_SPLIT_BATCH];
#pragma unroll
          for (int i = 0; i < U_SPLIT_BATCH; ++i) u[i] = src[t + 64 * (U_SPLIT_BATCH * h + i)];
#pragma unroll
          for (int i = 0; i < U_SPLIT_BATCH; ++i) {
            float4 l;
            l.x = u[i].x - __uint_as_float(__float_as_uint(u[i].x) & 0xffffe000u);
            l.y = u[i].y - __uint_as_float(__float_as_uint(u[i].y) & 0xffffe000u);
            l.z = u[i].z - __uint_as_float(__float_as_uint(u[i].z) & 0xffffe000u);
            l.w = u[i].w - __uint_as_float(__float_as_uint(u[i].w) & 0xffffe000u);
            lo[t + 64 * (U_SPLIT_BATCH * h + i)] = l;
          }
        }
#endif
        fence_proxy_async_smem();
        mbar_arrive(&conv[s]);
        if (++s == U_STAGES) { s = 0; ph ^= 1; }
      }
    }
    }
  } else {
    // drain + epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (its row quarter), columns half h
    const int q = warp & 3, h = (warp - 4) >> 2;
    int buf = 0;
    uint32_t tph = 0;  // phase bit of accumulator buffer b at bit b
    float inv_sig = 1.f;  // 2xFP16: the data scale 2^-e (exact), applied before `scale`
    if constexpr (F16) inv_sig = pow2f(-u_data_exp(a.amax, a.n_amax, a.amax_scale));
    float osig = 1.f;  // OUT16: the output's scale 2^e'
    if constexpr (OUT16) osig = pow2f(u_data_exp(a.amax, a.n_amax, a.out_scale16));
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const UItem ui = u_item<SPLIT>(a, it);
      const int mt = ui.mt, nt = ui.nt;
      const int b0 = 0, b1 = ui.hi - ui.lo;
      float acc[128];
#pragma unroll
      for (int c = 0; c < 128; ++c) acc[c] = 0.f;
      // OUT16: the multiplier of each of the warp's 128 columns, osig * scale * 2^-e_c (per-column source scales,
      // or the global 2^-e), loaded while the MMAs run and kept in the warp's shared-memory table (all lanes read
      // the same entry: broadcast).  Powers of two commute with the rounding, so (osig scale 2^-e) acc is
      // bit-identical to osig (scale (2^-e acc)).
      float4 cv = make_float4(1.f, 1.f, 1.f, 1.f);
      if constexpr (OUT16) {
        cv = a.cinv ? __ldg(reinterpret_cast<const float4*>(a.cinv + ui.nt * 256 + h * 128) + lane)
                    : make_float4(inv_sig, inv_sig, inv_sig, inv_sig);
        const float m = osig * a.scale;
        cv = make_float4(m * cv.x, m * cv.y, m * cv.z, m * cv.w);
      }
      for (int g0 = b0; g0 < b1; g0 += a.group) {
        mbar_wait(&tfull[buf], (tph >> buf) & 1u);
        tph ^= 1u << buf;
        tc_fence_after();
        const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + buf * 256 + h * 128;
#pragma unroll
        for (int c = 0; c < 128; c += 16) {
          float v[16];
          tmem_ld16(base + c, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[c + i] += v[i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        buf ^= 1;
      }
      // output: per 32-column chunk the warp's 32 x 32 block goes through its swizzled staging buffer and one
      // TMA store (or TMA add when accumulating); rows / columns outside the output are clipped by the TMA unit
      uint8_t* stg = sout + (warp - 4) * U_STAGE_OUT;
      float* mtab = reinterpret_cast<float*>(bars + 4 * U_STAGES + 8) + 128 * (warp - 4);  // OUT16: 512 B per warp
      const int r0 = (a.tile_mode == 0 ? mt * 128 + 32 * q
                                        : (2 * (mt / (a.tm_nz >> 6)) + (q >> 1)) * a.tm_nz + 64 * (mt % (a.tm_nz >> 6)) + 32 * (q & 1)) +
                     ui.kc * a.kc_rows;
      const int c0 = nt * 256 + h * 128;
      constexpr int CW = OUT16 ? 64 : 32;  // columns per store
#pragma unroll
      for (int c = 0; c < 128; c += CW) {
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
        if constexpr (OUT16) {  // fp16 hi / lo of 2^e' out: two 32 x 64 tiles, 128-byte rows, 128-byte swizzle
          if (c == 0) {  // the warp's multiplier table, written once per item (the previous item's reads are done)
            reinterpret_cast<float4*>(mtab)[lane] = cv;
            __syncwarp();
          }
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            uint32_t hw[4], lw[4];
            const float4 m0 = reinterpret_cast<const float4*>(mtab)[(c >> 2) + 2 * jj];
            const float4 m1 = reinterpret_cast<const float4*>(mtab)[(c >> 2) + 2 * jj + 1];
            const float ci[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float x0 = ci[2 * i] * acc[c + 8 * jj + 2 * i];
              const float x1 = ci[2 * i + 1] * acc[c + 8 * jj + 2 * i + 1];
              const __half2 hh = __floats2half2_rn(x0, x1);
              const float2 hf = __half22float2(hh);
              const __half2 ll = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
              hw[i] = *reinterpret_cast<const uint32_t*>(&hh);
              lw[i] = *reinterpret_cast<const uint32_t*>(&ll);
            }
            const int o = lane * 128 + ((jj ^ (lane & 7)) << 4);
            *reinterpret_cast<uint4*>(stg + o) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(stg + 4096 + o) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&out_map, c0 + c, r0, stg);
            tma_store_2d(&out_lo_map, c0 + c, r0, stg + 4096);
            bulk_commit();
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 v;
          if constexpr (F16)
            v = make_float4(a.scale * (inv_sig * acc[c + 4 * j]), a.scale * (inv_sig * acc[c + 4 * j + 1]),
                            a.scale * (inv_sig * acc[c + 4 * j + 2]), a.scale * (inv_sig * acc[c + 4 * j + 3]));
          else
            v = make_float4(a.scale * acc[c + 4 * j], a.scale * acc[c + 4 * j + 1], a.scale * acc[c + 4 * j + 2],
                            a.scale * acc[c + 4 * j + 3]);
          *reinterpret_cast<float4*>(stg + lane * 128 + ((j ^ (lane & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
#ifndef BAND_U_NO_EPI_WRITE
        if (lane == 0) {
          if (a.accumulate) tma_add_2d(&out_map, c0 + c, r0, stg);
          else tma_store_2d(&out_map, c0 + c, r0, stg);
          bulk_commit();
        }
#endif
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace lfm
