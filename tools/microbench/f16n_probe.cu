// kind::f16 MMA shapes with both operands K-major 64-byte swizzle (band_v's 2xFP16 adjoint: M128 N16 / N32):
// all-ones operands, one K=16 MMA per shape, D should be 16 everywhere.  One launch per shape (a fault stops there).
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include "tc_sm100.h"
using namespace lfm::tc;
__global__ void __launch_bounds__(128, 1) probe(int N, float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (8192 + 16384) / 2; i += 128) ((__half*)base)[i] = __float2half(1.f);
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_f16(128, N, 0, 0);
    mma_bf16_ss(tm, smem_desc(smem_u32(base), 16, 512, 4), smem_desc(smem_u32(base + 8192), 16, 512, 4), idesc, 0);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[8];
  tmem_ld_n<8>(tm + ((uint32_t)(32 * warp) << 16), v);
  D[tid] = v[0];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tm);
}
int main(int argc, char** argv) {
  const int N = atoi(argv[1]);
  float* d;
  cudaMalloc(&d, 512);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 + 16384 + 1024);
  probe<<<1, 128, 8192 + 16384 + 1024>>>(N, d);
  cudaError_t e = cudaDeviceSynchronize();
  float h[128];
  cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  printf("N %d: %s, D[0] %g D[127] %g\n", N, cudaGetErrorString(e), h[0], h[127]);
  return 0;
}
