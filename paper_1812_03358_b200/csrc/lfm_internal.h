// Internal structures of liblfm: host plan (fp64 build, fp32 device tables) and kernel launch
// descriptors.  Not part of the public ABI (include/lfm.h is).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/lfm.h"

namespace lfm {

// One separable axis of an affine ray map (s,u) -> (m00 s + m01 u + o0, m10 s + m11 u + o1), §2.1.
struct Affine {
  double m00, m01, m10, m11, o0, o1;
};

// One axis of an optical plane: n cells of width delta centred on c0, and X^{0p}.
struct Plane {
  int n;
  double delta;
  Affine X0;
  double c0;
};

// A family of banded 1D operator tables sharing the row count and padded tap count.
// Table m, row r: band start (first source cell), band length, taps weights (fp64 on the host,
// fp32 on the device; entries beyond `len` are zero).
// The device uses the ELL form: per row the exact non-zero list (count, source index, weight), padded
// to `ell` entries, stored [table][entry][row] so that lanes on consecutive rows coalesce.
struct BandFamily {
  int n_tables = 0, n_rows = 0, n_src = 0, taps = 0;
  std::vector<int32_t> start, len;
  std::vector<double> w64;
  int ell = 0;                       // padded entries per row (multiple of 4)
  std::vector<int32_t> cnt, eidx;    // [table][row], [table][entry][row]
  std::vector<double> ew64;          // [table][entry][row]
  int32_t* d_cnt = nullptr;
  int32_t* d_idx = nullptr;
  float* d_w = nullptr;
  // G4 form (rows grouped by 4): per group the union window [j0, j0+W) of source cells and W x 4
  // dense weights (row-interleaved), used when the family is the t side of an op (warp-uniform).
  int n_groups = 0, gmax = 0;
  std::vector<int32_t> g_j0, g_w, g_off;  // [table][group]
  std::vector<double> g_w64;              // flat, per table contiguous
  int32_t* d_g = nullptr;                 // int4 per [table][group]: j0, W, off, 0
  float* d_gw = nullptr;
  // MSEG form (built when want_mseg): per group a CSR list of segments, split at every all-zero run of
  // >= 2 source cells; segment = int4 {j0, W, off, 0}, weights W x 4 (row-interleaved) at off.
  int want_mseg = 0;
  std::vector<int32_t> m_off;              // [table*n_groups + g] .. +1 (size n_tables*n_groups + 1)
  std::vector<int32_t> m_seg;              // 4 ints per segment
  std::vector<double> m_w64;
  int32_t* d_moff = nullptr;
  int32_t* d_mseg = nullptr;
  float* d_mw = nullptr;
  // flat form of the MSEG lists (built with want_mseg): per group a list of (source row, 4 weights)
  // entries padded to a multiple of 4 with zero weights, so the kernel loop has no segment structure
  std::vector<int32_t> f_off, f_row;       // f_off: [table*n_groups + g] .. +1 in entries
  std::vector<double> f_w64;               // 4 per entry
  int32_t* d_foff = nullptr;
  int32_t* d_frow = nullptr;
  float* d_fw = nullptr;
  // tcgen05 form (band_u): per tile of 128 rows the union of the rows' supports cut into blocks of 16 source
  // cells; per block two 128 x 16 tf32 weight images (hi, lo) in the shared-memory layout the MMA reads
  std::vector<int32_t> u_off, u_k0;        // u_off[table * n_tiles + tile] .. +1 into blocks; u_k0[block]
  int u_mode = 0, u_nz = 0;                // tile composition (build_umma): 0 = 128 rows, 1 = 2 vt x 64 slices
  int u_ntiles = 0;                        // row tiles per table: ceil(n_rows/128) (mode 0), ceil(ny/2)*nz/64 (mode 1)
  std::vector<float> u_a;                  // 4096 floats per block
  int32_t* d_uoff = nullptr;
  int32_t* d_uk0 = nullptr;
  float* d_ua = nullptr;
  // 2xFP16 form of the same blocks (band_u_kernel<.., true>): per block the weights scaled by 2^u_wexp (exact) and
  // split w 2^e = hi + lo + O(2^-22 w 2^e), hi = rn_fp16(w 2^e), lo = rn_fp16(w 2^e - hi), each a 128 x 16 fp16 image
  // in the K-major 32-byte-swizzled layout (element (m, k) at byte m*32 + k*2 with bit 4 ^= bit 7): 4096 halves
  std::vector<uint16_t> u_h;
  int u_wexp = 0;                          // max |w| 2^u_wexp in [2^14, 2^15)
  float u_lsum = 0.f;                      // max over rows of sum |w| (fp32 weights): |out| <= u_lsum max |src|
  uint16_t* d_uh = nullptr;
  // the same with groups of 8 rows (weights 8 per source cell): half the source loads per FMA
  std::vector<int32_t> m8_off, m8_seg;
  std::vector<double> m8_w64;
  int32_t* d_m8off = nullptr;
  int32_t* d_m8seg = nullptr;
  float* d_m8w = nullptr;
  // density statistics (LFM_DEBUG): non-zeros, G4 slot columns, columns with any non-zero
  double st_nnz = 0, st_cols_g4 = 0, st_cols_nz = 0, st_msegs = 0, st_cols_m = 0;
};

// One summand of a separable banded sum: source plane at src_base + src_off, s/t table indices.
struct Term {
  long long src_off;
  int s_tab;
  int t_tab;
  float scale;
  int pad;
};

// Per (table, output tile): first source cell and width of the staged footprint (width 0 = empty).
struct Footprint {
  int32_t lo, width;
};
// Per (t-table, output tile_y): footprint plus the tile's block of G4 weights.
struct TileT {
  int32_t lo, width, woff, wlen;
};

// out[b] = out_scale * sum_{terms of b} scale * (B_s[s_tab] (x) B_t[t_tab]) src   (t-pass, s-pass)
struct SepOp {
  const BandFamily* fs = nullptr;  // rows = output s cells
  const BandFamily* ft = nullptr;  // rows = output t cells
  int n_os = 0, n_ot = 0, n_is = 0, n_it = 0, n_out = 0;
  float out_scale = 1.f;
  int ts = 128, tt = 64, nt = 256;  // output tile, threads per CTA
  int fs_max = 0, ft_max = 0;      // max source footprint per tile (s, t)
  std::vector<Term> terms;
  std::vector<int32_t> offs;       // n_out + 1
  Term* d_terms = nullptr;
  int32_t* d_offs = nullptr;
  int ntx = 0, nty = 0;            // output tiles along s, t
  int nb = 1;                      // terms staged per barrier
  int stage = 1;                   // stage the source footprint in smem (0: pass 1 reads L1/L2)
  int s_ident = 0;                 // the s family is the identity (pass 1 = copy into U)
  int kind = 0;                    // 0: sep_kernel,
                                   // 3: band_m_kernel (L2 gather over MSEG segments of ft)
                                   // 5: band_f_kernel (flat MSEG entry lists, L2 gather, deep unroll)
                                   // 8: band_u_kernel (tcgen05 kind::tf32 3xTF32, 128-row tiles, TMA, TMEM)
  long long src_pitch = 0;         // floats between source rows (0: n_is)
  long long out_pitch = 0;         // floats between output rows (0: n_os)
  long long out_stride = 0;        // floats between outputs b (0: n_os * n_ot)
  int tout = 0;                    // band_m only: write element (row, col) at col * out_pitch + row
  int mgrp = 4;                    // band_m only: rows per MSEG group (4 or 8)
  int chunk = 32;                  // (unused, kept in the tune-cache line format)
  int stages = 2;                  // band_m / band_f unroll; band_u drain group
  int wt_max = 0;                  // max G4 weight floats of one t tile
  int ws_max = 0;                  // max G4 weight floats of one s tile
  int nbuf = 2;                    // 2: double-buffered chunks, 1: one chunk per output
  TileT* d_fp_s = nullptr;         // [s-table][tile_x]
  TileT* d_fp_t = nullptr;         // [t-table][tile_y]
  double fma_alg = 0;              // sum over terms of nnz work (algorithmic)
};

// One shear pass of the rotation (eqn,rot,toeplitz): per line, first offset m_lo and taps weights.
struct ShearPass {
  int active = 0;
  int axis = 0;  // 0 = z-pass, 1 = x-pass, 2 = y-pass
  double c1 = 0, c2 = 0;
  int taps = 0, n_lines = 0;
  std::vector<int32_t> mlo[2];     // [fwd, adj]
  std::vector<double> w64[2];
  int32_t* d_mlo[2] = {nullptr, nullptr};
  float* d_w[2] = {nullptr, nullptr};
};

// tcgen05 s-pass tables (band_v.cuh): per item (slice n, N-tile) the K blocks and the N x BK hi/lo images
struct VTab {
  int N = 0, n_nt = 0, BK = 16;
  float lsum = 0.f;  // max over rows (output columns) of sum |w|: |U| <= lsum max |x| (the 2xFP16 data scale)
  // 2xFP16 images (BK 32 only): 2^wexp w split into fp16 hi + lo, same K-major layout with 64-byte rows (64-byte
  // swizzle), hi N x BK then lo N x BK per block
  std::vector<uint16_t> h16;
  int wexp = 0;
  uint16_t* d_h16 = nullptr;
  std::vector<int32_t> off, k0;
  std::vector<float> img;
  int32_t* d_off = nullptr;
  int32_t* d_k0 = nullptr;
  float* d_img = nullptr;
};

// Per-view ops restricted to one view subset (sec,subset): compact field slots j <-> views S[j].
// When the subset is a tensor product S = S_s x {all k_t} (M | K_s, reading R5's k = k_t K_s + k_s), the
// subset operator is also K-collapsible: C^S_{s,n} = (K/|S|) sum_{k_s in S_s} S_ks B_ks,n, the t composite being
// the full one -- then `collapsed` is set and the subset runs on the collapsed two-pass path with these s tables.
struct ViewOps {
  SepOp fwd_s1, fwd_s3, adj_s3, adj_s1;
  int n_views = 0;
  int collapsed = 0;
  BandFamily cfs, cas;   // subset s composites (forward C^S_s,n and its transpose), K/|S| included
  VTab vf, va;           // their band_v tables
};

// Term tau >= 1 of a non-separable lenslet stage (hexagonal layout / circular apertures, reading R12): its collapsed
// composites, the slice-interleaved t families with their tcgen05 images, the band_v tables and the two t-pass ops.
struct Component {
  BandFamily cf[2], ca[2], ca1n, cf1n;
  VTab vf, va;
  SepOp fwd_c2, adj_c1;
};

struct CameraPlan {
  lfm_camera cam;
  lfm_info info;
  BandFamily s1f[2], s1a[2], s3f[2], s3a[2], cf[2], ca[2];
  // A_forward / A_adjoint ops, per path
  SepOp fwd_s1, fwd_s3, adj_s3, adj_s1;   // per-view path
  SepOp fwd_c, adj_c1, adj_c2;            // collapsed path (adjoint in two passes: t then s)
  SepOp fwd_c1, fwd_c2;                   // collapsed forward in two passes: s (U_n for all n), then t
  int fwd_split = 0;                      // 1: forward uses fwd_c1 + fwd_c2 (chosen by the autotuner)
  SepOp fwd_p1, adj_a2;                   // transposed s passes (band_m with transposed output)
  int fwd_t = 0;                          // forward s pass: 0 sep, 1 transpose x + fwd_p1, 2 spass_fwd, 3 band_v (autotuner)
  int adj_t = 0;                          // adjoint s pass: 0 sep, 1 transpose Z + adj_a2, 2 spass_adj, 3 band_v (autotuner)
  BandFamily id_s, id_t, id_vt;           // identity row maps used by the two-pass adjoint/forward
  BandFamily ca1n, cf1n;                  // slice-interleaved collapsed t families (rows (vt,n) / sources (vt,n))
  // lf_transport ops (output b = n*K + k for slice-indexed families)
  SepOp xp_s1f, xp_s1a, xp_s3f, xp_s3a;
  ShearPass rot[3];                       // application order z, x, y (x^r = E^y E^x E^z x)
  int has_perm = 0;                       // quarter-turn relabelling applied before the shears (reading R7)
  int perm_axis[2][3], perm_sign[2][3];   // [fwd: P, adj: P^T] source axis and sign per output axis
  std::vector<ViewOps> subs;              // view-subset ops (lfm_geometry.n_subsets > 1)
  double scal[8];                         // c1, c3, Va, Vmu_or_Vd, dz_r, V_axis..., see plan.cpp
  int spa_vta = 8;                        // voxel rows per CTA of the direct adjoint s pass (4 or 8, autotuned)
  // tcgen05 s passes (band_v.cuh): forward (from cf[0]) and adjoint (from ca[0]) tables
  using VTab = lfm::VTab;
  VTab vf, va;
  size_t ws_rot = 0, ws_fields = 0, ws_z = 0;
  int n_terms = 1;                        // separable terms of the lenslet stage (1: separable geometry)
  std::vector<Component> comps;           // terms 1 .. n_terms - 1
};

}  // namespace lfm

struct lfm_plan_s {
  int device = 0;
  int n_subsets = 0;
  lfm_volume vol;
  std::vector<lfm::CameraPlan> cams;
};

namespace lfm {
// plan.cpp (host fp64)
void ell_footprint(const BandFamily& f, int tab, int tile, int t, int& lo, int& width);
void g4_tile(const BandFamily& f, int tab, int tile, int t, int& lo, int& width, int& woff, int& wlen);
size_t sep_smem(const SepOp& op, int nb);
void fill_sep_geometry(SepOp& op);
bool sep_choose_tile(SepOp& op);
lfm_status autotune_camera(CameraPlan& cp, std::string& err);
lfm_status build_camera(const lfm_volume& vol, const lfm_camera& cam, int n_subsets, CameraPlan& out,
                        std::string& err);
lfm_status prepare_subsets(CameraPlan& cp, std::string& err);
uint16_t f2h_rn(float x);  // fp32 -> fp16 bits, round to nearest even (|x| < 65520)
float h2f(uint16_t h);
// kernels.cu
lfm_status upload_camera(CameraPlan& cp, std::string& err);
void free_camera(CameraPlan& cp);
// Pre-split source of the 2xFP16 band_u form: fp16 arrays hi, lo (same shape and pitch as the fp32 source) holding
// 2^e src = hi + lo, e = u_data_exp(max of the LFM_AMAX_SLOTS partial maxima `amax` x amax_scale) as their producer
// computed it (band_v forward: maxima of x^r times the s composite's row-sum bound; split16_kernel: maxima of the
// source itself).  hi == nullptr: the 3xTF32 form on the fp32 source.
constexpr int LFM_AMAX_SLOTS = 256;  // partial maxima slots in the workspace (>= CTAs of any launch writing them)
struct F16Src {
  const uint16_t* hi = nullptr;
  const uint16_t* lo = nullptr;
  const float* amax = nullptr;
  float amax_scale = 1.f;
  const float* cinv = nullptr;  // per-column data scales 2^-e_c (k_split16_cols) instead of the global 2^-e
  // optional fp16 output (the adjoint's Z for band_v's 2xFP16 form): hi / lo arrays shaped like the fp32 output,
  // 2^e' out with e' = u_data_exp(amax, out_scale16); not with split-K or accumulation
  uint16_t* out_hi = nullptr;
  uint16_t* out_lo = nullptr;
  float out_scale16 = 1.f;
};
lfm_status launch_sep(const SepOp& op, const float* src, float* out, int b0, int n_out, int accumulate,
                      void* stream, std::string& err, int out_r0 = 0, int out_r1 = -1, int win_r0 = 0,
                      int win_r1 = -1, int out_c0 = 0, int out_c1 = -1, float* part = nullptr,
                      size_t part_bytes = 0, F16Src h16 = F16Src());
lfm_status k_transpose(const float* in, float* out, int B, int R, int C, long long in_bs, long long in_pitch,
                       long long out_bs, long long out_pitch, void* stream, std::string& err);
lfm_status k_spass_fwd(const CameraPlan& cp, const float* x, float* U, void* stream, std::string& err);
// amax != nullptr: U is written as fp16 hi (U reinterpreted as uint16_t*, nd*nz*ny halves) then lo (the next
// nd*nz*ny halves) of 2^e U with e from the partial maxima of |x| (amax_kernel) and T.lsum -- the 2xFP16 t pass input
// x16 != nullptr too (and BK 32 fp16 tables): 2xFP16 input, x16 = fp16 hi (n_vox) then lo of 2^e x (split16_kernel
// with the same maxima)
// rinv != nullptr: x16 was split with per-row scales (split16_rows_kernel), rinv[n ny + vt] = 2^-e_row
lfm_status k_vpass_fwd(const CameraPlan& cp, const VTab& T, const float* x, float* U, void* stream, std::string& err,
                       int c0 = 0, int c1 = -1, const float* amax = nullptr, const uint16_t* x16 = nullptr,
                       const float* rinv = nullptr);
lfm_status k_split16_rows(const float* src, int rows, int len, float* part, float* rinv, uint16_t* hi, uint16_t* lo,
                          void* stream, std::string& err);
// column-scaled split of a rows x cols source (pitch cols): hi / lo of 2^e_c src, cinv[c] = 2^-e_c (1 for the padding
// columns [cols, cols_pad)), per-CTA maxima of |src| into part -- the adjoint t pass's input (one kernel)
lfm_status k_split16_cols(const float* src, int rows, int cols, int cols_pad, float* part, float* cinv, uint16_t* hi,
                          uint16_t* lo, void* stream, std::string& err);
// the same split of the PWLS residual r = w (Ax - gamma[cam] y) computed on the load (r itself never stored)
lfm_status k_split16_cols_residual(const float* Ax, const float* y, const float* w, const double* gamma, int cam,
                                   int rows, int cols, int cols_pad, float* part, float* cinv, uint16_t* hi, uint16_t* lo,
                                   void* stream, std::string& err);
// LFM_AMAX_SLOTS partial maxima of |src[0, n)| into part (one kernel)
lfm_status k_amax(const float* src, long long n, float* part, void* stream, std::string& err);
// fp16 hi / lo of 2^e src over n floats (e from the partial maxima `amax` of src), for the 2xFP16 band_u form
lfm_status k_split16(const float* src, long long n, const float* amax, uint16_t* hi, uint16_t* lo, void* stream,
                     std::string& err);
// amax != nullptr (and BK 32, N 16 fp16 tables): Z is fp16 hi then lo of 2^e Z, e = u_data_exp(amax, in_scale)
// (band_u adjoint's fp16 output); otherwise fp32 Z
lfm_status k_vpass_adj(const CameraPlan& cp, const VTab& T, const float* Z, float* out, int accumulate, void* stream,
                       std::string& err, int c0 = 0, int c1 = -1, const float* amax = nullptr, float in_scale = 1.f);
// whether k_vpass_adj can take an fp16 Z for table T
inline bool vpass_adj_in16(const VTab& T) { return T.d_h16 && (T.BK == 32 || T.BK == 64) && T.N == 16; }
lfm_status k_spass_adj(const CameraPlan& cp, const float* Z, float* out, int accumulate, void* stream, std::string& err);
lfm_status k_permute(const float* in, float* out, int nx, int ny, int nz, const int* axis, const int* sign,
                     int accumulate, void* stream, std::string& err);
}  // namespace lfm
