// Probe of tcgen05 kind::f16 (fp16 inputs, fp32 accumulate) for the 2xFP16 band_u variant: (1) operand layouts
// -- A (weights) K-major 32-byte swizzle or no swizzle, K = 16 (32 bytes per row); B (data) MN-major 128-byte
// swizzle, 16 K rows x 256 N -- checked against a CPU product of the same fp16 values, (2) the 3-product split
// D = A_lo B_hi + A_hi B_lo + A_hi B_hi of fp32 operands vs the fp64 product, (3) MMA throughput.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1812_03358_b200/csrc \
//        tools/microbench/f16_probe.cu -o /tmp/f16_probe -lcuda && /tmp/f16_probe
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_sm100.h"

using namespace lfm::tc;

constexpr int M = 128, N = 256, BK = 16;

// A (M x 16, K-major): SW32: row m at m*32 bytes, bit 4 ^= bit 7; NONE: [m/8][k/8][m%8][16 B]
__host__ __device__ inline uint32_t a_off(int m, int k, int lay) {
  if (lay == 6) {
    uint32_t off = (uint32_t)(m * 32 + k * 2);
    return off ^ (((off >> 7) & 1u) << 4);
  }
  return (uint32_t)((m / 8) * 256 + (k / 8) * 128 + (m % 8) * 16 + (k % 8) * 2);
}
// B (16 x N, MN-major SW128): N atom g = n/64 at g*16*128, k row at k*128, bits [4,7) ^= bits [7,10)
__host__ __device__ inline uint32_t b_off(int k, int n) {
  uint32_t off = (uint32_t)((n / 64) * BK * 128 + k * 128 + (n % 64) * 2);
  return off ^ (((off >> 7) & 7u) << 4);
}

__host__ __device__ constexpr uint32_t idesc_f16(int M_, int N_, int a_mn, int b_mn) {
  return (1u << 4) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N_ >> 3) << 17) |
         ((uint32_t)(M_ >> 4) << 24);
}

// D = sum over nprod products of A_p B_p (each one K=16 MMA), repeated `chain` times; D out [M][N]
__global__ void __launch_bounds__(128, 1) probe(const __half* A, const __half* B, int nprod, int chain, float* D,
                                                long long* clk, int alay, uint32_t albo, uint32_t asbo, uint32_t blbo,
                                                uint32_t bsbo) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int p = 0; p < nprod; ++p) {
    uint8_t* sA = base + p * 4096;
    uint8_t* sB = base + 16384 + p * 8192;
    for (int i = tid; i < M * BK; i += 128) *(__half*)(sA + a_off(i / BK, i % BK, alay)) = A[p * M * BK + i];
    for (int i = tid; i < BK * N; i += 128) *(__half*)(sB + b_off(i / N, i % N)) = B[p * BK * N + i];
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  constexpr uint32_t IDESC = idesc_f16(M, N, 0, 1);
  if (tid == 0) {
    const long long t0 = clock64();
    for (int c = 0; c < chain; ++c)
      for (int p = 0; p < nprod; ++p)
        mma_bf16_ss(tm, smem_desc(smem_u32(base + p * 4096), albo, asbo, alay),
                    smem_desc(smem_u32(base + 16384 + p * 8192), blbo, bsbo, 2), IDESC, (c | p) != 0);
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    clk[0] = clock64() - t0;
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + c, v);
    for (int i = 0; i < 32; ++i) D[(size_t)tid * N + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

int main() {
  srand(1);
  std::vector<float> Af(M * BK), Bf(BK * N);
  for (auto& v : Af) v = (float)rand() / RAND_MAX - 0.3f;
  for (auto& v : Bf) v = (float)rand() / RAND_MAX - 0.3f;
  // hi/lo split of fp32 operands into fp16 pairs (values of order 1: no scaling needed here)
  std::vector<__half> Ah(M * BK), Al(M * BK), Bh(BK * N), Bl(BK * N);
  for (int i = 0; i < M * BK; ++i) {
    Ah[i] = __float2half_rn(Af[i]);
    Al[i] = __float2half_rn(Af[i] - __half2float(Ah[i]));
  }
  for (int i = 0; i < BK * N; ++i) {
    Bh[i] = __float2half_rn(Bf[i]);
    Bl[i] = __float2half_rn(Bf[i] - __half2float(Bh[i]));
  }
  __half *dA, *dB;
  float* dD;
  long long* dclk;
  cudaMalloc(&dA, 3 * M * BK * 2);
  cudaMalloc(&dB, 3 * BK * N * 2);
  cudaMalloc(&dD, M * N * 4);
  cudaMalloc(&dclk, 16);
  const size_t smem = 16384 + 3 * 8192 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  std::vector<float> D(M * N);
  auto run = [&](const std::vector<__half>& a, const std::vector<__half>& b, int nprod, int chain, int alay,
                 uint32_t albo, uint32_t asbo, uint32_t blbo, uint32_t bsbo) {
    cudaMemcpy(dA, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
    probe<<<1, 128, smem>>>(dA, dB, nprod, chain, dD, dclk, alay, albo, asbo, blbo, bsbo);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long long c;
    cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
    return c;
  };
  // (1) layouts: one product of the fp16 values, vs the CPU product of the same values
  struct V { int alay; uint32_t albo, asbo, blbo, bsbo; } vs[] = {
      {6, 16, 256, 2048, 1024}, {6, 16, 256, 1024, 2048}, {0, 128, 256, 2048, 1024}, {0, 256, 128, 2048, 1024}};
  for (auto& v : vs) {
    run(Ah, Bh, 1, 1, v.alay, v.albo, v.asbo, v.blbo, v.bsbo);
    double e = 0, mx = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < BK; ++k) s += (double)__half2float(Ah[m * BK + k]) * __half2float(Bh[k * N + n]);
        e = fmax(e, fabs(D[m * N + n] - s));
        mx = fmax(mx, fabs(s));
      }
    printf("layout A lay %d lbo %u sbo %u | B lbo %u sbo %u: max|D - ref| = %.3e (max|ref| %.3f)\n", v.alay, v.albo,
           v.asbo, v.blbo, v.bsbo, e, mx);
  }
  // (2) 3-product split vs fp64 of the fp32 operands
  {
    std::vector<__half> a3(3 * M * BK), b3(3 * BK * N);
    for (int i = 0; i < M * BK; ++i) a3[i] = Al[i], a3[M * BK + i] = Ah[i], a3[2 * M * BK + i] = Ah[i];
    for (int i = 0; i < BK * N; ++i) b3[i] = Bh[i], b3[BK * N + i] = Bl[i], b3[2 * BK * N + i] = Bh[i];
    run(a3, b3, 3, 1, 6, 16, 256, 2048, 1024);
    double e = 0, mx = 0, e32 = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        float s32 = 0.f;
        for (int k = 0; k < BK; ++k) s += (double)Af[m * BK + k] * Bf[k * N + n], s32 += Af[m * BK + k] * Bf[k * N + n];
        e = fmax(e, fabs(D[m * N + n] - s));
        e32 = fmax(e32, fabs((double)s32 - s));
        mx = fmax(mx, fabs(s));
      }
    printf("2xFP16 split (3 products): max|D - fp64| = %.3e, fp32 FMA chain %.3e (max|ref| %.3f)\n", e, e32, mx);
    long long c = run(a3, b3, 3, 1000, 6, 16, 256, 2048, 1024);
    printf("throughput: %lld clk for %d MMAs (M128 N256 K16 f16) -> %.1f clk/MMA\n", c, 3000, (double)c / 3000);
  }
  return 0;
}
