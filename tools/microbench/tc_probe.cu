// Probe of tcgen05 kind::tf32 on this B200: (1) operand layouts used by band_u (A K-major SW64 from a
// pre-swizzled image, B MN-major SW128), (2) how fp32 inputs are reduced to tf32 (truncation or
// rounding), (3) how the TMEM accumulator rounds when MMAs are chained, (4) raw MMA throughput.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1812_03358_b200/csrc \
//        tools/microbench/tc_probe.cu -o /tmp/tc_probe -lcuda && /tmp/tc_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tc_sm100.h"

using namespace lfm::tc;

constexpr int M = 128, N = 256, BK = 16;

__host__ __device__ inline uint32_t swz64(uint32_t off) { return off ^ (((off >> 7) & 3u) << 4); }
__host__ __device__ inline uint32_t swz128(uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); }
// A (M x BK, K-major, SW64): row m at m*64 bytes
__host__ __device__ inline uint32_t a_off(int m, int k) { return swz64((uint32_t)(m * 64 + k * 4)); }
// B (BK x N, MN-major, SW128): N-group g = n/32 at g*BK*128, k row at k*128
__host__ __device__ inline uint32_t swz128a32(uint32_t off) { return off ^ (((off >> 7) & 3u) << 5); }
__host__ __device__ inline uint32_t b_off(int k, int n) { return swz128a32((uint32_t)((n / 32) * BK * 128 + k * 128 + (n % 32) * 4)); }

// D = A0 B0 (fresh), then `chain` more MMAs D += A1 B1 (each the 2 k-steps of the block); D out [M][N]
__global__ void __launch_bounds__(128, 1) probe(const float* A0, const float* B0, const float* A1, const float* B1,
                                                int chain, float* D, long long* clk, uint32_t idesc_in) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  uint8_t* sA0 = base;             // 8 KB each
  uint8_t* sA1 = base + 8192;
  uint8_t* sB0 = base + 16384;     // 16 KB each
  uint8_t* sB1 = base + 32768;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * BK; i += 128) {
    const int m = i / BK, k = i % BK;
    *(float*)(sA0 + a_off(m, k)) = A0[i];
    *(float*)(sA1 + a_off(m, k)) = A1[i];
  }
  for (int i = tid; i < BK * N; i += 128) {
    const int k = i / N, n = i % N;
    *(float*)(sB0 + b_off(k, n)) = B0[i];
    *(float*)(sB1 + b_off(k, n)) = B1[i];
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
  const uint32_t idesc = idesc_in;
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int j = 0; j < BK / 8; ++j)
      mma_tf32_ss(tm, smem_desc(smem_u32(sA0) + 32 * j, 16, 512, 4), smem_desc(smem_u32(sB0) + 1024 * j, BK * 128, 512, 1),
                  idesc, j > 0);
    for (int c = 0; c < chain; ++c)
      for (int j = 0; j < BK / 8; ++j)
        mma_tf32_ss(tm, smem_desc(smem_u32(sA1) + 32 * j, 16, 512, 4),
                    smem_desc(smem_u32(sB1) + 1024 * j, BK * 128, 512, 1), idesc, 1);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  if (tid == 0) {
    t1 = clock64();
    clk[0] = t1 - t0;
  }
  tc_fence_after();
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + c, v);
    for (int i = 0; i < 32; ++i) D[(size_t)tid * N + c + i] = v[i];
  }
  if (clk[1] == 7) {  // TMEM store/load round trip at column 300
    uint32_t a = tm + ((uint32_t)(32 * warp) << 16) + 300;
    float w = 1.0f + tid;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a), "r"(__float_as_uint(w)));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (tid % 40 == 0) printf("roundtrip tid %d: wrote %g read %g\n", tid, w, __uint_as_float(r));
    if (tid == 0) printf("smem A0 word0 %g (A0[0] %g) idesc %x descA %llx descB %llx\n", *(float*)sA0, A0[0], idesc,
        (unsigned long long)smem_desc(smem_u32(sA0), 16, 512, 4), (unsigned long long)smem_desc(smem_u32(sB0), BK * 128, 1024, 2));
  }
  if (clk[1] == 7) {  // debug scan of all 512 columns, lane 0..127
    for (int c = 0; c < 512; c += 32) {
      float v[32];
      tmem_ld32(tm + ((uint32_t)(32 * warp) << 16) + c, v);
      int nz = 0;
      for (int i = 0; i < 32; ++i) nz += v[i] != 0.f;
      if (nz && (tid % 32 == 0)) printf("tid %d cols %d..: %d nonzero, v0 %g\n", tid, c, nz, v[0]);
    }
    if (tid == 0) printf("tmem base %x\n", tm);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}


__global__ void __launch_bounds__(128, 1) probe_bf16(float* D, uint32_t idesc, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 49152 / 4; i += 128) ((uint32_t*)base)[i] = 0x3F803F80u;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    uint64_t a = smem_desc(smem_u32(base), 16, 1024, 2), b = smem_desc(smem_u32(base) + 16384, lbo, sbo, lay);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tm), "l"(a), "l"(b), "r"(idesc), "r"(0));
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[32];
  tmem_ld32(tm + ((uint32_t)(32 * warp) << 16), v);
  D[tid] = v[0];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

static float trunc_tf32(float v) { uint32_t u; memcpy(&u, &v, 4); u &= 0xffffe000u; memcpy(&v, &u, 4); return v; }
static float rna_tf32(float v) { uint32_t u; memcpy(&u, &v, 4); u += 0x1000u; u &= 0xffffe000u; memcpy(&v, &u, 4); return v; }

int main() {
  std::vector<float> A0(M * BK), B0(BK * N), A1(M * BK, 0.f), B1(BK * N, 0.f), D(M * N);
  srand(1);
  for (auto& v : A0) v = (float)rand() / RAND_MAX - 0.3f;
  for (auto& v : B0) v = (float)rand() / RAND_MAX - 0.3f;
  float *dA0, *dB0, *dA1, *dB1, *dD;
  long long* dclk;
  cudaMalloc(&dA0, A0.size() * 4); cudaMalloc(&dB0, B0.size() * 4); cudaMalloc(&dA1, A1.size() * 4);
  cudaMalloc(&dB1, B1.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dclk, 16); { long long d[2] = {0, 7}; cudaMemcpy(dclk, d, 16, cudaMemcpyHostToDevice); }
  const size_t smem = 49152 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  uint32_t g_idesc = idesc_tf32(M, N, 0, 1);
  auto run = [&](int chain) {
    cudaMemcpy(dA0, A0.data(), A0.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB0, B0.data(), B0.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dA1, A1.data(), A1.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB1, B1.data(), B1.size() * 4, cudaMemcpyHostToDevice);
    probe<<<1, 128, smem>>>(dA0, dB0, dA1, dB1, chain, dD, dclk, g_idesc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); exit(1); }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long long c; cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
    return c;
  };
  {
    cudaFuncSetAttribute(probe_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    auto idb = [](int M_, int N_, int a_mn, int b_mn) { return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N_ >> 3) << 17) | ((uint32_t)(M_ >> 4) << 24); };
    struct V { int amn, bmn; uint32_t lbo, sbo, lay; } vs[] = {{0,0,16,1024,2},{0,1,2048,1024,2},{0,1,1024,2048,2},{0,1,16,1024,0},{0,1,4096,1024,2}};
    for (auto& v : vs) {
      probe_bf16<<<1, 128, smem>>>(dD, idb(128, 256, v.amn, v.bmn), v.lbo, v.sbo, v.lay);
      cudaDeviceSynchronize();
      float h[128]; cudaMemcpy(h, dD, 512, cudaMemcpyDeviceToHost);
      printf("bf16 ones a_mn %d b_mn %d lbo %u sbo %u lay %u: D[0] %g D[127] %g (expect 16)\n", v.amn, v.bmn, v.lbo, v.sbo, v.lay, h[0], h[127]);
    }
  }
  // (0): all ones -> D = BK everywhere for any consistent layout
  {
    std::vector<float> a0 = A0, b0 = B0;
    std::fill(A0.begin(), A0.end(), 1.f); std::fill(B0.begin(), B0.end(), 1.f);
    run(0);
    printf("ones test: D[0] %g D[last] %g (expect %d)\n", D[0], D[M * N - 1], BK);
    uint32_t variants[4] = {idesc_tf32(M, N, 0, 0), idesc_tf32(M, N, 1, 1), idesc_tf32(64, N, 0, 1), idesc_tf32(M, 128, 0, 1)};
    for (int v = 0; v < 4; ++v) {
      g_idesc = variants[v];
      run(0);
      printf("ones test variant %d idesc %x: D[0] %g D[last] %g\n", v, g_idesc, D[0], D[M * N - 1]);
    }
    g_idesc = idesc_tf32(M, N, 0, 1);
    A0 = a0; B0 = b0;
  }
  // (1)+(2): layouts and input conversion
  run(0);
  double et = 0, er = 0, ef = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double st = 0, sr = 0, sf = 0;
      for (int k = 0; k < BK; ++k) {
        st += (double)trunc_tf32(A0[m * BK + k]) * trunc_tf32(B0[k * N + n]);
        sr += (double)rna_tf32(A0[m * BK + k]) * rna_tf32(B0[k * N + n]);
        sf += (double)A0[m * BK + k] * B0[k * N + n];
      }
      et = fmax(et, fabs(D[m * N + n] - st));
      er = fmax(er, fabs(D[m * N + n] - sr));
      ef = fmax(ef, fabs(D[m * N + n] - sf));
    }
  printf("D[0..3] %g %g %g %g\n", D[0], D[1], D[2], D[3]);
  printf("layout/input test: max|D - trunc-tf32 ref| = %.3e, |D - rna-tf32 ref| = %.3e, |D - fp32 ref| = %.3e\n", et, er, ef);
  // (3): accumulator rounding.  D0 = 1 (A0 = e_0 column, B0 row 0 = 1); each chained MMA adds 0.75 ulp(1)
  std::fill(A0.begin(), A0.end(), 0.f);
  std::fill(B0.begin(), B0.end(), 0.f);
  for (int m = 0; m < M; ++m) A0[m * BK] = 1.f, A1[m * BK] = 1.f;
  for (int n = 0; n < N; ++n) B0[n] = 1.f, B1[n] = 0.75f * ldexpf(1.f, -23);
  run(50);
  printf("accumulate test (100 adds of +0.75 ulp): D-1 = %.3e ulp  (RN: 100, RZ: 0)\n", (D[0] - 1.0) / ldexp(1.0, -23));
  for (int n = 0; n < N; ++n) B1[n] = -0.75f * ldexpf(1.f, -23);
  run(50);
  printf("accumulate test (100 adds of -0.75 ulp): D-1 = %.3e ulp(1)  (RN: about -100/2.., RZ: -50 (ulp below 1 is half))\n",
         (D[0] - 1.0) / ldexp(1.0, -23));
  // (4): throughput, one CTA: 2 k-steps per chained block
  std::fill(B1.begin(), B1.end(), 1e-3f);
  long long c = run(2000);
  printf("throughput: %lld clk for %d MMAs (M128 N256 K8) -> %.1f clk/MMA\n", c, 2 * 2001, (double)c / (2 * 2001));
  return 0;
}
