// Standalone check + timing of band_u_kernel (paper_1812_03358_b200/csrc/band_u.cuh) on random banded
// operators: out = scale * C src, compared with an fp64 host product.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1812_03358_b200/csrc \
//        tools/microbench/band_u_test.cu -o tools/microbench/band_u_test
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "band_u.cuh"

using namespace lfm;

static float tf32_rn(float v) { uint32_t u; memcpy(&u, &v, 4); u += 0x1000u; u &= 0xffffe000u; memcpy(&v, &u, 4); return v; }
static uint32_t swz64(uint32_t off) { return off ^ (((off >> 7) & 3u) << 4); }

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Problem {
  int R, K, N;
  std::vector<std::vector<std::pair<int, float>>> rows;  // per row: (k, w)
};

static Problem make_problem(int R, int K, int N, bool wide, unsigned seed) {
  std::mt19937 g(seed);
  std::uniform_real_distribution<float> U(0.f, 1.f);
  Problem p{R, K, N, {}};
  p.rows.resize(R);
  for (int r = 0; r < R; ++r) {
    if (!wide) {
      int c = (int)((long long)r * K / R) + (int)(g() % 7) - 3;
      int len = 1 + g() % 8;
      for (int q = 0; q < len; ++q)
        if (c + q >= 0 && c + q < K) p.rows[r].push_back({c + q, U(g)});
    } else if (R > 4096) {  // adjoint-t-pass-like: tile window of ~208 source rows, rows of 54 taps
      const int t = r / 128;
      const int w0 = (int)((long long)t * (K - 208) / std::max(1, R / 128 - 1));
      std::vector<float> w(208, 0.f);
      int c = (int)(g() % (208 - 54));
      for (int q = 0; q < 54; ++q) w[c + q] = U(g);
      for (int q = 0; q < 208; ++q)
        if (w[q] != 0.f) p.rows[r].push_back({w0 + q, w[q]});
    } else {  // forward-t-pass-like: tile window of ~1900 source rows, 8 runs of 52 per row
      const int t = r / 128;
      const int w0 = (int)((long long)t * (K - 1922) / std::max(1, R / 128 - 1));
      std::vector<float> w(1922, 0.f);
      for (int run = 0; run < 8; ++run) {
        int c = (int)(g() % (1922 - 52));
        for (int q = 0; q < 52; ++q) w[c + q] = U(g);
      }
      for (int q = 0; q < 1922; ++q)
        if (w[q] != 0.f) p.rows[r].push_back({w0 + q, w[q]});
    }
  }
  return p;
}

int main(int argc, char** argv) {
  EncodeFn encode = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &qr);
  if (!encode) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  cudaFuncSetAttribute(band_u_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  struct Case { int R, K, N; bool wide; int group; int reps; };
  Case cases[] = {{300, 200, 600, false, 2, 0}, {300, 200, 600, false, 1000, 0}, {2048, 16384, 2048, true, 8, 20},
                  {2048, 16384, 2048, true, 4, 20}, {16384, 2048, 2048, true, 4, 20}};
  for (const Case& cs : cases) {
    Problem p = make_problem(cs.R, cs.K, cs.N, cs.wide, 7);
    // blocks
    const int n_mt = (p.R + 127) / 128;
    std::vector<int> off(n_mt + 1, 0), k0;
    std::vector<float> A;
    std::vector<std::vector<float>> dense;
    for (int mt = 0; mt < n_mt; ++mt) {
      off[mt] = (int)k0.size();
      std::vector<char> any(p.K, 0);
      for (int r = mt * 128; r < std::min(p.R, mt * 128 + 128); ++r)
        for (auto& e : p.rows[r]) any[e.first] = 1;
      std::vector<int> starts;
      for (int k = 0; k < p.K; ++k)
        if (any[k] && (starts.empty() || k >= starts.back() + 16)) starts.push_back(k);
      for (int s : starts) {
        k0.push_back(s);
        std::vector<float> img(4096, 0.f);
        for (int m = 0; m < 128; ++m) {
          const int r = mt * 128 + m;
          if (r >= p.R) continue;
          for (auto& e : p.rows[r]) {
            const int k = e.first - s;
            if (k < 0 || k >= 16) continue;
            const float hi = tf32_rn(e.second), lo = tf32_rn(e.second - hi);
            const uint32_t o = swz64((uint32_t)(m * 64 + k * 4)) / 4;
            img[o] += hi;  // rows hold distinct k, so += is a store
            img[2048 + o] += lo;
          }
        }
        A.insert(A.end(), img.begin(), img.end());
      }
    }
    off[n_mt] = (int)k0.size();
    std::vector<float> src((size_t)p.K * p.N), out((size_t)p.R * p.N);
    std::mt19937 g(3);
    std::normal_distribution<float> Nd(0.f, 1.f);
    for (auto& v : src) v = std::fabs(Nd(g)) + 0.1f;
    float *dA, *dsrc, *dout;
    int *doff, *dk0;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dsrc, src.size() * 4); cudaMalloc(&dout, out.size() * 4);
    cudaMalloc(&doff, off.size() * 4); cudaMalloc(&dk0, k0.size() * 4 + 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dsrc, src.data(), src.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(doff, off.data(), off.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dk0, k0.data(), k0.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t gdim[2] = {(cuuint64_t)p.N, (cuuint64_t)p.K};
    cuuint64_t gstr[1] = {(cuuint64_t)p.N * 4};
    cuuint32_t box[2] = {32, 16}, es[2] = {1, 1};
    CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dsrc, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
    CUtensorMap omap;
    {
      cuuint64_t od[2] = {(cuuint64_t)p.N, (cuuint64_t)p.R};
      cuuint64_t os[1] = {(cuuint64_t)p.N * 4};
      cuuint32_t ob[2] = {32, 32};
      cr = encode(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dout, od, os, ob, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) { printf("encode out failed %d\n", (int)cr); return 1; }
    }
    UArgs a;
    a.A = dA; a.blk_off = doff; a.blk_k0 = dk0; a.out = dout; a.out_pitch = p.N; a.n_rows = p.R; a.n_cols = p.N;
    a.mt0 = 0; a.n_mt = n_mt; a.n_nt = (p.N + 255) / 256; a.k_shift = 0; a.k_end = p.K; a.windowed = 0; a.group = cs.group; a.scale = 1.f;
    a.accumulate = 0;
    a.tile_mode = 0;
    a.tm_nz = 0;
    const int grid = std::min(nsm, n_mt * a.n_nt);
    band_u_kernel<<<grid, U_THREADS, U_SMEM>>>(map, omap, a);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    double emax = 0, rmax = 0, bias = 0;
    long long nb = 0;
    for (int r = 0; r < p.R; r += (cs.wide ? 7 : 1))
      for (int c = 0; c < p.N; ++c) {
        double ref = 0;
        for (auto& en : p.rows[r]) ref += (double)en.second * src[(size_t)en.first * p.N + c];
        emax = std::max(emax, std::fabs(out[(size_t)r * p.N + c] - ref));
        rmax = std::max(rmax, std::fabs(ref));
        if (ref != 0) { bias += (out[(size_t)r * p.N + c] - ref) / ref; ++nb; }
      }
    double nnz = 0;
    for (auto& row : p.rows) nnz += row.size();
    printf("R %d K %d N %d group %d: blocks %zu (density %.3f)  max|err|/max|ref| = %.3e  mean rel bias %.2e\n", p.R, p.K,
           p.N, cs.group, k0.size(), nnz / (k0.size() * 128.0 * 16), emax / rmax, nb ? bias / nb : 0.0);
    if (cs.reps) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int i = 0; i < cs.reps; ++i) band_u_kernel<<<grid, U_THREADS, U_SMEM>>>(map, omap, a);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= cs.reps;
      const double mma_fma = (double)k0.size() * 128 * 16 * p.N * 3;
      printf("   %.4f ms  alg %.2f TFLOP/s  tensor %.1f%% of %d SMs x 2048 tf32 FMA/clk @1.965 GHz\n", ms,
             2 * nnz * p.N / ms / 1e9, 100 * mma_fma / (ms * 1e-3) / (nsm * 2048.0 * 1.965e9), nsm);
    }
    cudaFree(dA); cudaFree(dsrc); cudaFree(dout); cudaFree(doff); cudaFree(dk0);
  }
  return 0;
}
