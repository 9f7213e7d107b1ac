// Kernel launchers (kernels.cu) used by the C-ABI layer (api.cu).
#pragma once
#include <string>

#include "lfm_internal.h"

namespace lfm {
extern thread_local int g_launches;
lfm_status launch_shear(const ShearPass& sp, int dir, const float* in, float* out, int nx, int ny, int nz,
                        int accumulate, void* stream, std::string& err);
lfm_status k_copy_scale(const float* in, float* out, long long n, float scale, int acc, void* s, std::string& err);
lfm_status k_fill(float* out, long long n, float v, void* s, std::string& err);
lfm_status k_mul(const float* a, const float* b, float* out, long long n, void* s, std::string& err);
lfm_status k_stats(const float* Ax, const float* y, const float* w, long long n, double* part, double* out, void* s,
                   std::string& err);
lfm_status k_gains(const double* stats, int n_cam, double* gamma, int* flag, void* s, std::string& err);
lfm_status k_residual(const float* Ax, const float* y, const float* w, const double* gamma, int cam, float* r,
                      long long n, double* part, double* cost, int cost_acc, void* s, std::string& err);
lfm_status k_reg26(const float* x, float* grad, int nx, int ny, int nz, float beta, float nu, double* part,
                   double* cost, void* s, std::string& err);
lfm_status k_fista(float* x, float* z, const float* grad, const float* d, long long n, float tau, void* s,
                   std::string& err);
lfm_status k_majoriser_finish(float* d, long long n, float add, void* s, std::string& err);
}  // namespace lfm
