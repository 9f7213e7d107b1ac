// TMA load throughput per SM on B200 for the shapes the t-pass kernels use: (a) 2D tensor boxes of 16 rows x 128 B
// from rows 4 KB apart (band_u's source tiles), (b) the same boxes over rows 128 B apart (contiguous 2 KB), (c) 1D
// bulk copies of 8 KB contiguous images.  148 CTAs, one producer thread each, a ring of STAGES x 24 KB, no consumer
// work: reports bytes per cycle per SM.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1812_03358_b200/csrc \
//        tools/microbench/tma_rate.cu -o /tmp/tma_rate -lcuda && /tmp/tma_rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "tc_sm100.h"

using namespace lfm::tc;
constexpr int STAGES = 8, STAGE = 24576, ITERS = 2000;

// mode 0: 12 tensor boxes (64 x 16 fp16) per stage from the strided map; 1: same from the contiguous map;
// 2: 3 bulk copies of 8 KB; 3: 3 3D boxes (64 x 16 x 4: 4 column groups of 64 in one box, the group stride 128 B
// overlapping the row stride) from the strided data; 4: 3 2D boxes of 64 rows x 128 B (8 KB contiguous, no
// swizzle: a verbatim copy of a pre-laid-out image, as band_u's weight images)
__global__ void __launch_bounds__(128, 1) rate(const __grid_constant__ CUtensorMap m_str, const __grid_constant__ CUtensorMap m_con,
                                               const __grid_constant__ CUtensorMap m_3d,
                                               const __grid_constant__ CUtensorMap m_img,
                                               const uint8_t* src, long long src_bytes, int mode, long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long t0 = clock64();
  uint32_t ph = 0;
  int s = 0;
  for (int it = 0; it < ITERS; ++it) {
    if (it >= STAGES) mbar_wait(&full[s], ph ^ 1);
    uint8_t* st = base + s * STAGE;
    mbar_arrive_expect_tx(&full[s], STAGE);
    const int blk = (blockIdx.x * 7919 + it * 104729) & 1023;  // pseudo-random block of rows / images
    if (mode == 4) {
      for (int j = 0; j < 3; ++j) tma_load_2d(st + j * 8192, &m_img, 0, ((blk * 3 + j) * 64) % (16384 * 32), &full[s]);
    } else if (mode == 3) {
      for (int j = 0; j < 3; ++j) tma_load_3d(st + j * 8192, &m_3d, 0, (blk * 48 + j * 16) % 16384, 0, &full[s]);
    } else if (mode == 2) {
      for (int j = 0; j < 3; ++j)
        bulk_g2s(st + j * 8192, src + ((long long)(blk * 3 + j) * 8192) % (src_bytes - 8192), 8192, &full[s]);
    } else {
      const CUtensorMap* m = mode == 0 ? &m_str : &m_con;
      for (int j = 0; j < 12; ++j) tma_load_2d(st + j * 2048, m, (j % 4) * 64, (blk * 48 + (j / 4) * 16) % 16384, &full[s]);
    }
    if (++s == STAGES) { s = 0; ph ^= 1; }
  }
  for (int it = ITERS - STAGES; it < ITERS; ++it) mbar_wait(&full[it % STAGES], (it / STAGES) & 1);  // drain
  clk[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long bytes = 64ll << 20;
  uint8_t* d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  long long* dclk;
  cudaMalloc(&dclk, 148 * 8);
  EncodeFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap ms, mc;
  cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
  {  // rows of 2048 halves (4 KB), 16384 rows
    cuuint64_t gd[2] = {2048, 16384}, gs[1] = {4096};
    enc(&ms, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {  // rows of 64 halves (128 B): a box is 2 KB contiguous
    cuuint64_t gd[2] = {64, 16384 * 32}, gs[1] = {128};
    enc(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  CUtensorMap m3;
  {  // the strided data as (64 columns, rows, column groups): box 64 x 16 x 4 = 8 KB, [group][row][64] in shared memory
    cuuint64_t gd[3] = {64, 16384, 32}, gs[2] = {4096, 128};
    cuuint32_t b3[3] = {64, 16, 4}, e3[3] = {1, 1, 1};
    CUresult r = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, d, gd, gs, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("3D map with overlapping group stride: encode %s (%d)\n", r == CUDA_SUCCESS ? "ok" : "FAILED", (int)r);
    if (r != CUDA_SUCCESS) m3 = ms;
  }
  CUtensorMap mi;
  {  // 8 KB images as rows of 128 B, box 64 rows, no swizzle
    cuuint64_t gd[2] = {64, 16384 * 32}, gs[1] = {128};
    cuuint32_t bi[2] = {64, 64}, ei[2] = {1, 1};
    enc(&mi, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, gd, gs, bi, ei, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  const int smem = STAGES * STAGE + 1024;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[5] = {"tensor boxes 16 x 128 B, rows 4 KB apart", "tensor boxes 16 x 128 B, contiguous", "bulk 8 KB",
                          "3D boxes 4 x 16 x 128 B, rows 4 KB apart", "2D boxes 64 x 128 B (8 KB image), no swizzle"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 5; ++mode) {
      rate<<<148, 128, smem>>>(ms, mc, m3, mi, d, bytes, mode, dclk);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<long long> c(148);
      cudaMemcpy(c.data(), dclk, 148 * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      double avg = 0;
      for (long long v : c) mx = v > mx ? v : mx, avg += v / 148.0;
      if (rep) printf("%-45s: %.1f B/cycle/SM (avg CTA), %.1f (slowest); %.0f cycles per 24 KB stage\n", names[mode],
                      (double)ITERS * STAGE / avg, (double)ITERS * STAGE / mx, avg / ITERS);
    }
  return 0;
}
