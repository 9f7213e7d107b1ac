// liblfm plan builder: host fp64, compiled with -ffp-contract=off (no FMA contraction) so the
// integer band tables follow a documented expression order (reading Z21).
//
// What it computes, per camera (P = PAPER.md line):
//  * optics chain per axis (§2.1): T_d, R_f(c), composition, inverse;
//  * rotation Theta = D S_z S_x S_y (eqn,rot,decomp P:1127-1135) in closed form, relabelled
//    voxel sizes Delta/D, and per-line shear tables (eqn,rot,toeplitz P:1186-1198);
//  * per (axis, angular index, slice) the 1D transport factors of eqn,xport,int
//    as banded tables: weights = (1/|b_q|) int_{cell j} Trap(s - c_i) ds, the closed form of the
//    missing tab,pillbox / tab,dirac, evaluated in fp64, rounded once to fp32;
//  * adjoint tables from the opposite transport B^{qp} (closed form from the other side), used as
//    the scaled forward operation;
//  * the lenslet stage S_k = sum_mu B^{mu a}_k M_mu with rasterised square apertures (P:915-927,
//    P:1011-1024), and the K-collapsed composite C_n = sum_k S_k B^{a q_n}_k (exact re-association).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <map>
#include <vector>

#include "lfm_internal.h"

namespace lfm {

static Affine translate(double d) { return {1.0, d, 0.0, 1.0, 0.0, 0.0}; }
static Affine lens(double f, double c) { return {1.0, 0.0, -1.0 / f, 1.0, 0.0, c / f}; }

static Affine compose(const Affine& a, const Affine& b) {  // a o b
  Affine r;
  r.m00 = a.m00 * b.m00 + a.m01 * b.m10;
  r.m01 = a.m00 * b.m01 + a.m01 * b.m11;
  r.m10 = a.m10 * b.m00 + a.m11 * b.m10;
  r.m11 = a.m10 * b.m01 + a.m11 * b.m11;
  r.o0 = a.m00 * b.o0 + a.m01 * b.o1 + a.o0;
  r.o1 = a.m10 * b.o0 + a.m11 * b.o1 + a.o1;
  return r;
}

static bool invert(const Affine& a, Affine& out) {
  double det = a.m00 * a.m11 - a.m01 * a.m10;
  if (std::fabs(det) <= 1e-12) return false;
  double i00 = a.m11 / det;
  double i01 = -a.m01 / det;
  double i10 = -a.m10 / det;
  double i11 = a.m00 / det;
  out.m00 = i00; out.m01 = i01; out.m10 = i10; out.m11 = i11;
  out.o0 = -(i00 * a.o0 + i01 * a.o1);
  out.o1 = -(i10 * a.o0 + i11 * a.o1);
  return true;
}

static double centre(const Plane& p, int i) { return p.c0 + ((double)i - (p.n - 1) * 0.5) * p.delta; }

struct Kernel1D {  // one row family of a transport q -> p at angular centre s_k
  double lam, mu, nu, W, w, H, bq_abs;
  double sk;
};

// s_p = lam*s_q + mu*s_0 + nu (substituting u -> s_0 in eqn,xport,ip); trapezoid (W, w, H).
static lfm_status make_kernel(const Plane& src, const Plane& dst, double s_k, double d0, int basis,
                              Kernel1D& k, std::string& err) {
  Affine inv;
  if (!invert(dst.X0, inv)) { err = "singular X^{0p} block"; return LFM_E_SINGULAR; }
  Affine Xpq = compose(inv, src.X0);  // X^{pq} = (X^{0p})^{-1} o X^{0q}
  double P = Xpq.m00, Q = Xpq.m01, o_pq = Xpq.o0;
  double a_q = src.X0.m00, b_q = src.X0.m01, o_q = src.X0.o0;
  if (b_q == 0.0) { err = "source plane on the angular plane (b_q = 0)"; return LFM_E_DEGENERATE; }
  k.lam = P - Q * a_q / b_q;
  k.mu = Q / b_q;
  k.nu = o_pq - Q * o_q / b_q;
  if (k.lam == 0.0) { err = "destination conjugate to the angular plane (lambda = 0)"; return LFM_E_DEGENERATE; }
  double al = std::fabs(k.lam);
  double dp = dst.delta;
  if (basis == LFM_DIRAC) {
    k.W = dp / (2.0 * al);
    k.w = dp / (2.0 * al);
    k.H = d0;
  } else {
    double am = std::fabs(k.mu);
    k.W = (d0 * am + dp) / (2.0 * al);
    k.w = std::fabs(d0 * am - dp) / (2.0 * al);
    k.H = (am == 0.0) ? d0 : std::min(d0, dp / am);
  }
  k.bq_abs = std::fabs(b_q);
  k.sk = s_k;
  return LFM_OK;
}

static double trap_value(double x, double W, double w, double H) {
  double ax = std::fabs(x);
  if (ax <= w) return H;
  if (ax < W) return H * (W - ax) / (W - w);
  return 0.0;
}

// Exact integral of the trapezoid over [lo, hi]: midpoint rule on each linear piece.
static double trap_integral(double lo, double hi, double W, double w, double H) {
  const double p0s[3] = {-W, -w, w};
  const double p1s[3] = {-w, w, W};
  double total = 0.0;
  for (int q = 0; q < 3; ++q) {
    double p0 = p0s[q], p1 = p1s[q];
    if (p1 <= p0) continue;
    double l = std::max(lo, p0);
    double h = std::min(hi, p1);
    if (h > l) total += (h - l) * trap_value(0.5 * (l + h), W, w, H);
  }
  return total;
}

// Row i of the transport: centre c_i on the source plane and the analytic band (reading Z21).
static void row_band(const Plane& src, const Plane& dst, const Kernel1D& k, int i, double& c, int& lo, int& hi) {
  c = (centre(dst, i) - k.nu - k.mu * k.sk) / k.lam;
  double dq = src.delta;
  double s0 = src.c0 + (0.0 - (src.n - 1) * 0.5) * dq;
  double flo = std::floor((c - k.W - s0 - 0.5 * dq) / dq) + 1.0;
  double fhi = std::ceil((c + k.W - s0 + 0.5 * dq) / dq) - 1.0;
  flo = std::max(flo, 0.0);
  fhi = std::min(fhi, (double)(src.n - 1));
  if (fhi < flo) { lo = 0; hi = -1; return; }
  lo = (int)flo;
  hi = (int)fhi;
}

static double entry(const Plane& src, const Kernel1D& k, double c, int j) {
  double sj = centre(src, j);
  return trap_integral(sj - 0.5 * src.delta - c, sj + 0.5 * src.delta - c, k.W, k.w, k.H) / k.bq_abs;
}

// A sparse row: band [lo, lo+len) with weights (zeros allowed inside).
struct Row {
  int lo = 0, len = 0;
  std::vector<double> w;
};

static lfm_status transport_rows(const Plane& src, const Plane& dst, double s_k, double d0, int basis,
                                 std::vector<Row>& rows, std::string& err) {
  Kernel1D k;
  lfm_status st = make_kernel(src, dst, s_k, d0, basis, k, err);
  if (st != LFM_OK) return st;
  rows.assign(dst.n, Row());
  for (int i = 0; i < dst.n; ++i) {
    double c;
    int lo, hi;
    row_band(src, dst, k, i, c, lo, hi);
    Row& r = rows[i];
    if (hi < lo) continue;
    r.lo = lo;
    r.len = hi - lo + 1;
    r.w.resize(r.len);
    for (int j = lo; j <= hi; ++j) r.w[j - lo] = entry(src, k, c, j);
  }
  return LFM_OK;
}

static double basis_volume(const Plane& p, double d0) { return p.delta * d0 / std::fabs(p.X0.m01); }

// Append a table (n_rows rows) to a family; taps is fixed later (max len).
static void family_init(BandFamily& f, int n_tables, int n_rows, int n_src) {
  f.n_tables = n_tables;
  f.n_rows = n_rows;
  f.n_src = n_src;
  f.taps = 0;
  f.start.assign((size_t)n_tables * n_rows, 0);
  f.len.assign((size_t)n_tables * n_rows, 0);
}

// Build the ELL form (exact non-zero list per row) from the band rows.
static void build_ell(BandFamily& f) {
  int mx = 1;
  f.cnt.assign((size_t)f.n_tables * f.n_rows, 0);
  for (int m = 0; m < f.n_tables; ++m)
    for (int r = 0; r < f.n_rows; ++r) {
      size_t idx = (size_t)m * f.n_rows + r;
      int c = 0;
      for (int q = 0; q < f.len[idx]; ++q) c += f.w64[idx * f.taps + q] != 0.0;
      f.cnt[idx] = c;
      mx = std::max(mx, c);
    }
  f.ell = (mx + 3) / 4 * 4;
  size_t per = (size_t)f.ell * f.n_rows;
  f.eidx.assign((size_t)f.n_tables * per, 0);
  f.ew64.assign((size_t)f.n_tables * per, 0.0);
  for (int m = 0; m < f.n_tables; ++m)
    for (int r = 0; r < f.n_rows; ++r) {
      size_t idx = (size_t)m * f.n_rows + r;
      int e = 0;
      int first = f.len[idx] ? f.start[idx] : 0;
      for (int q = 0; q < f.len[idx]; ++q) {
        double w = f.w64[idx * f.taps + q];
        if (w == 0.0) continue;
        f.eidx[m * per + (size_t)e * f.n_rows + r] = f.start[idx] + q;
        f.ew64[m * per + (size_t)e * f.n_rows + r] = w;
        ++e;
      }
      for (; e < f.ell; ++e) f.eidx[m * per + (size_t)e * f.n_rows + r] = first;  // zero-weight padding
    }
  // G4 form: groups of 4 consecutive rows; the union window of their bands is split at its longest
  // all-zero run (if any) into at most two segments; dense row-interleaved weights per segment
  f.n_groups = (f.n_rows + 3) / 4;
  size_t ng = (size_t)f.n_tables * f.n_groups;
  f.g_j0.assign(2 * ng, 0);
  f.g_w.assign(2 * ng, 0);
  f.g_off.assign(2 * ng, 0);
  f.g_w64.clear();
  f.gmax = 0;
  f.m_seg.clear();
  f.m_w64.clear();
  if (f.want_mseg) f.m_off.assign(ng + 1, 0);
  std::vector<double> dense;
  for (int m = 0; m < f.n_tables; ++m)
    for (int g = 0; g < f.n_groups; ++g) {
      int lo = 1 << 30, hi = -1;
      for (int q = 0; q < 4; ++q) {
        int r = 4 * g + q;
        if (r >= f.n_rows) break;
        size_t idx = (size_t)m * f.n_rows + r;
        if (!f.len[idx]) continue;
        lo = std::min(lo, (int)f.start[idx]);
        hi = std::max(hi, (int)(f.start[idx] + f.len[idx]));
      }
      size_t gi = (size_t)m * f.n_groups + g;
      f.g_off[2 * gi] = f.g_off[2 * gi + 1] = (int)f.g_w64.size();
      if (f.want_mseg) f.m_off[gi] = (int)(f.m_seg.size() / 4);
      if (hi < 0) continue;
      const int W = hi - lo;
      dense.assign((size_t)W * 4, 0.0);
      for (int q = 0; q < 4; ++q) {
        int r = 4 * g + q;
        if (r >= f.n_rows) break;
        size_t idx = (size_t)m * f.n_rows + r;
        for (int e = 0; e < f.len[idx]; ++e)
          dense[(size_t)(f.start[idx] + e - lo) * 4 + q] = f.w64[idx * f.taps + e];
      }
      // longest run of all-zero columns strictly inside the window
      int best_a = -1, best_len = 0;
      for (int p = 0; p < W;) {
        bool z = dense[4 * p] == 0.0 && dense[4 * p + 1] == 0.0 && dense[4 * p + 2] == 0.0 && dense[4 * p + 3] == 0.0;
        if (!z) { ++p; continue; }
        int a = p;
        while (p < W && dense[4 * p] == 0.0 && dense[4 * p + 1] == 0.0 && dense[4 * p + 2] == 0.0 && dense[4 * p + 3] == 0.0) ++p;
        if (a > 0 && p < W && p - a > best_len) { best_len = p - a; best_a = a; }
      }
      int segs[2][2] = {{0, W}, {0, 0}};  // [start, end) within the window
      if (best_len > 0) {
        segs[0][1] = best_a;
        segs[1][0] = best_a + best_len;
        segs[1][1] = W;
      }
      for (int sgi = 0; sgi < 2; ++sgi) {
        int a = segs[sgi][0], b = segs[sgi][1];
        f.g_j0[2 * gi + sgi] = lo + a;
        f.g_w[2 * gi + sgi] = b - a;
        f.g_off[2 * gi + sgi] = (int)f.g_w64.size();
        for (int p = a; p < b; ++p)
          for (int q = 0; q < 4; ++q) f.g_w64.push_back(dense[4 * p + q]);
      }
      f.gmax = std::max(f.gmax, W);
      for (int p = 0; p < W; ++p) {
        bool z = dense[4 * p] == 0.0 && dense[4 * p + 1] == 0.0 && dense[4 * p + 2] == 0.0 && dense[4 * p + 3] == 0.0;
        f.st_cols_nz += !z;
        for (int q = 0; q < 4; ++q) f.st_nnz += dense[4 * p + q] != 0.0;
      }
      f.st_cols_g4 += segs[0][1] - segs[0][0] + segs[1][1] - segs[1][0];
      // multi-segment form (MSEG): split the window at every all-zero run of >= 2 columns
      {
        int p = 0;
        while (p < W) {
          while (p < W && dense[4 * p] == 0.0 && dense[4 * p + 1] == 0.0 && dense[4 * p + 2] == 0.0 &&
                 dense[4 * p + 3] == 0.0)
            ++p;
          if (p >= W) break;
          int a = p, last = p;
          while (p < W) {
            bool z = dense[4 * p] == 0.0 && dense[4 * p + 1] == 0.0 && dense[4 * p + 2] == 0.0 && dense[4 * p + 3] == 0.0;
            if (!z) { last = p; ++p; continue; }
            int zs = p;
            while (p < W && dense[4 * p] == 0.0 && dense[4 * p + 1] == 0.0 && dense[4 * p + 2] == 0.0 &&
                   dense[4 * p + 3] == 0.0)
              ++p;
            if (p - zs >= 2 || p >= W) break;
          }
          f.st_msegs += 1;
          f.st_cols_m += last - a + 1;
          if (f.want_mseg) {
            f.m_seg.push_back(lo + a);
            f.m_seg.push_back(last - a + 1);
            f.m_seg.push_back((int)f.m_w64.size());
            f.m_seg.push_back(0);
            for (int c = a; c <= last; ++c)
              for (int q = 0; q < 4; ++q) f.m_w64.push_back(dense[4 * c + q]);
          }
        }
      }
    }
  if (f.want_mseg) {
    f.m_off[ng] = (int)(f.m_seg.size() / 4);
    // flat form: one entry per MSEG column, each group padded to a multiple of 4 entries
    f.f_off.assign(ng + 1, 0);
    f.f_row.clear();
    f.f_w64.clear();
    for (size_t gi = 0; gi < ng; ++gi) {
      f.f_off[gi] = (int)f.f_row.size();
      int last = 0;
      for (int sg = f.m_off[gi]; sg < f.m_off[gi + 1]; ++sg) {
        const int j0 = f.m_seg[4 * (size_t)sg], w = f.m_seg[4 * (size_t)sg + 1], wo = f.m_seg[4 * (size_t)sg + 2];
        for (int p = 0; p < w; ++p) {
          f.f_row.push_back(j0 + p);
          for (int q = 0; q < 4; ++q) f.f_w64.push_back(f.m_w64[wo + 4 * (size_t)p + q]);
          last = j0 + p;
        }
      }
      while (f.f_row.size() % 4) {
        f.f_row.push_back(last);
        for (int q = 0; q < 4; ++q) f.f_w64.push_back(0.0);
      }
    }
    f.f_off[ng] = (int)f.f_row.size();
  }
}

// Union window of the G4 groups of output tile t (rows [t*tile, (t+1)*tile)), and its weight block.
void g4_tile(const BandFamily& f, int tab, int tile, int t, int& lo, int& width, int& woff, int& wlen) {
  int g0 = t * tile / 4, g1 = std::min(f.n_groups, (t + 1) * tile / 4);
  int mn = 1 << 30, mx = -1;
  for (int g = g0; g < g1; ++g)
    for (int sgi = 0; sgi < 2; ++sgi) {
      size_t gi = 2 * ((size_t)tab * f.n_groups + g) + sgi;
      if (!f.g_w[gi]) continue;
      mn = std::min(mn, (int)f.g_j0[gi]);
      mx = std::max(mx, (int)(f.g_j0[gi] + f.g_w[gi]));
    }
  woff = g0 < f.n_groups ? f.g_off[2 * ((size_t)tab * f.n_groups + g0)] : 0;
  int end = (g1 < f.n_groups) ? f.g_off[2 * ((size_t)tab * f.n_groups + g1)]
                              : (tab + 1 < f.n_tables ? f.g_off[2 * ((size_t)(tab + 1) * f.n_groups)] : (int)f.g_w64.size());
  wlen = end - woff;
  if (mx < 0) { lo = 0; width = 0; return; }
  lo = mn;
  width = mx - mn;
}

struct FamilyBuilder {
  BandFamily& f;
  std::vector<std::vector<Row>> tabs;
  explicit FamilyBuilder(BandFamily& fam) : f(fam) {}
  void finish() {
    int taps = 1;
    for (auto& t : tabs)
      for (auto& r : t) taps = std::max(taps, r.len);
    f.taps = taps;
    f.w64.assign((size_t)f.n_tables * f.n_rows * taps, 0.0);
    for (int m = 0; m < f.n_tables; ++m)
      for (int r = 0; r < f.n_rows; ++r) {
        const Row& row = tabs[m][r];
        size_t idx = (size_t)m * f.n_rows + r;
        f.start[idx] = row.len ? row.lo : 0;
        f.len[idx] = row.len;
        for (int q = 0; q < row.len; ++q) f.w64[idx * taps + q] = row.w[q];
      }
    tabs.clear();
    build_ell(f);
  }
};

// tf32 value of an fp32 (round to nearest, ties away from zero, 10 explicit mantissa bits; the low 13 bits
// cleared), as cvt.rna.tf32.f32 does on the device.
static float tf32_round(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u += 0x1000u;
  u &= 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// tcgen05 form of a one-table family (band_u, band_u.cuh): tiles of 128 rows; the union of the rows'
// non-zero source cells covered by the fewest blocks of 16 consecutive cells (greedy); per block the fp32
// weights (one rounding from fp64) split as w = hi + lo + O(2^-22 w), hi = rn_tf32(w), lo = rn_tf32(w - hi),
// each a 128 x 16 image in the tensor core's K-major 64-byte-swizzled shared-memory layout: element (m, k) at
// byte m*64 + k*4 with bits [4,6) XOR bits [7,9).
// Tile composition: mode 0 = 128 consecutive rows; mode 1 (rows-by-slice families, rows r = vt*nz + n with
// nz % 64 == 0) = 2 consecutive voxel rows x 64 consecutive slices, whose supports overlap more (block density
// 0.287 vs 0.251 for 1 x 128 at 128^3).  Tile row m -> table row (-1 = none).
static int umma_row(const BandFamily& f, int t, int m) {
  if (f.u_mode == 0) {
    const int r = 128 * t + m;
    return r < f.n_rows ? r : -1;
  }
  const int per = f.u_nz / 64, p = t / per, hh = t % per;
  const int vt = 2 * p + (m >> 6), n = 64 * hh + (m & 63);
  const int r = vt * f.u_nz + n;
  return r < f.n_rows ? r : -1;
}

// fp32 -> fp16 bits, round to nearest even (normal and subnormal; |x| < 65520 assumed, as the callers scale to
// below 2^15), and back
uint16_t f2h_rn(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  const uint32_t sign = (u >> 16) & 0x8000u;
  u &= 0x7fffffffu;
  if (u < 0x38800000u) {  // below 2^-14: subnormal fp16, value m 2^-24 with m = rn_even(|x| 2^24) (exact product)
    float a;
    std::memcpy(&a, &u, 4);
    return (uint16_t)(sign | (uint32_t)std::nearbyint((double)a * 16777216.0));
  }
  const uint32_t r = (u + 0xfffu + ((u >> 13) & 1u)) >> 13;  // mantissa rounded to 10 bits (carry into exponent)
  return (uint16_t)(sign | (r - ((127u - 15u) << 10)));
}
float h2f(uint16_t h) {
  const int e = (h >> 10) & 31, m = h & 1023;
  const double v = e == 0 ? std::ldexp((double)m, -24) : std::ldexp(1.0 + m / 1024.0, e - 15);
  return (float)((h & 0x8000) ? -v : v);
}

static void build_umma(BandFamily& f) {
  // mode 1 pairs voxel rows: an odd ny leaves a last tile with one voxel row (its other half reads as none)
  const int nt = f.u_mode == 0 ? (f.n_rows + 127) / 128 : ((f.n_rows / f.u_nz + 1) / 2) * (f.u_nz / 64);
  f.u_ntiles = nt;
  f.u_off.assign((size_t)f.n_tables * nt + 1, 0);
  f.u_k0.clear();
  f.u_a.clear();
  std::vector<char> any;
  for (int m = 0; m < f.n_tables; ++m)
    for (int t = 0; t < nt; ++t) {
      f.u_off[(size_t)m * nt + t] = (int)f.u_k0.size();
      int lo = 1 << 30, hi = -1;
      for (int mm = 0; mm < 128; ++mm) {
        const int r = umma_row(f, t, mm);
        if (r < 0) continue;
        size_t idx = (size_t)m * f.n_rows + r;
        if (!f.len[idx]) continue;
        lo = std::min(lo, (int)f.start[idx]);
        hi = std::max(hi, (int)(f.start[idx] + f.len[idx]));
      }
      if (hi < 0) continue;
      any.assign(hi - lo, 0);
      for (int mm = 0; mm < 128; ++mm) {
        const int r = umma_row(f, t, mm);
        if (r < 0) continue;
        size_t idx = (size_t)m * f.n_rows + r;
        for (int e = 0; e < f.len[idx]; ++e)
          if (f.w64[idx * f.taps + e] != 0.0) any[f.start[idx] + e - lo] = 1;
      }
      std::vector<int> starts;
      for (int p = 0; p < hi - lo; ++p)
        if (any[p] && (starts.empty() || p >= starts.back() + 16)) starts.push_back(p);
      for (int a0 : starts) {
        const int k0 = lo + a0;
        f.u_k0.push_back(k0);
        const size_t base = f.u_a.size();
        f.u_a.resize(base + 4096, 0.f);
        for (int mm = 0; mm < 128; ++mm) {
          const int r = umma_row(f, t, mm);
          if (r < 0) continue;
          size_t idx = (size_t)m * f.n_rows + r;
          for (int k = 0; k < 16; ++k) {
            const int e = k0 + k - f.start[idx];
            if (e < 0 || e >= f.len[idx]) continue;
            const float w = (float)f.w64[idx * f.taps + e];
            const float wh = tf32_round(w), wl = tf32_round(w - wh);
            uint32_t off = (uint32_t)(mm * 64 + k * 4);
            off ^= ((off >> 7) & 3u) << 4;
            f.u_a[base + off / 4] = wh;
            f.u_a[base + 2048 + off / 4] = wl;
          }
        }
      }
    }
  f.u_off[(size_t)f.n_tables * nt] = (int)f.u_k0.size();
  // 2xFP16 images: w 2^e split into fp16 hi + lo, e so that max |w| 2^e lies in [2^14, 2^15)
  float wmax = 0.f;
  double lsum = 0;
  for (size_t idx = 0; idx < (size_t)f.n_tables * f.n_rows; ++idx) {
    double r = 0;
    for (int e = 0; e < f.len[idx]; ++e) {
      wmax = std::max(wmax, std::fabs((float)f.w64[idx * f.taps + e]));
      r += std::fabs((double)(float)f.w64[idx * f.taps + e]);
    }
    lsum = std::max(lsum, r);
  }
  f.u_lsum = (float)(lsum * (1.0 + 1e-6));
  int ex = 0;
  if (wmax > 0.f) std::frexp((double)wmax * (1.0 + 1e-6), &ex);
  f.u_wexp = wmax > 0.f ? 15 - ex : 0;
  const size_t nb = f.u_k0.size();
  f.u_h.assign(nb * 4096, 0);
  for (int m = 0; m < f.n_tables; ++m)
    for (int t = 0; t < nt; ++t)
      for (int b = f.u_off[(size_t)m * nt + t]; b < f.u_off[(size_t)m * nt + t + 1]; ++b) {
        const int k0 = f.u_k0[b];
        for (int mm = 0; mm < 128; ++mm) {
          const int r = umma_row(f, t, mm);
          if (r < 0) continue;
          const size_t idx = (size_t)m * f.n_rows + r;
          for (int k = 0; k < 16; ++k) {
            const int e = k0 + k - f.start[idx];
            if (e < 0 || e >= f.len[idx]) continue;
            const float w = (float)std::ldexp((double)(float)f.w64[idx * f.taps + e], f.u_wexp);  // exact
            const uint16_t wh = f2h_rn(w), wl = f2h_rn(w - h2f(wh));
            uint32_t off = (uint32_t)(mm * 32 + k * 2);
            off ^= ((off >> 7) & 1u) << 4;
            f.u_h[(size_t)b * 4096 + off / 2] = wh;
            f.u_h[(size_t)b * 4096 + 2048 + off / 2] = wl;
          }
        }
      }
}

// MSEG form with groups of 8 rows (segments split at zero runs >= 2 source cells, weights 8 per cell).
static void build_mseg8(BandFamily& f) {
  const int G = 8;
  const int ng = (f.n_rows + G - 1) / G;
  f.m8_off.assign((size_t)f.n_tables * ng + 1, 0);
  f.m8_seg.clear();
  f.m8_w64.clear();
  std::vector<double> dense;
  for (int m = 0; m < f.n_tables; ++m)
    for (int g = 0; g < ng; ++g) {
      f.m8_off[(size_t)m * ng + g] = (int)(f.m8_seg.size() / 4);
      int lo = 1 << 30, hi = -1;
      for (int r = G * g; r < std::min(f.n_rows, G * g + G); ++r) {
        size_t idx = (size_t)m * f.n_rows + r;
        if (!f.len[idx]) continue;
        lo = std::min(lo, (int)f.start[idx]);
        hi = std::max(hi, (int)(f.start[idx] + f.len[idx]));
      }
      if (hi < 0) continue;
      const int W = hi - lo;
      dense.assign((size_t)W * G, 0.0);
      for (int r = G * g; r < std::min(f.n_rows, G * g + G); ++r) {
        size_t idx = (size_t)m * f.n_rows + r;
        for (int e = 0; e < f.len[idx]; ++e) dense[(size_t)(f.start[idx] + e - lo) * G + (r - G * g)] = f.w64[idx * f.taps + e];
      }
      auto zero = [&](int c) {
        for (int q = 0; q < G; ++q)
          if (dense[(size_t)c * G + q] != 0.0) return false;
        return true;
      };
      int p = 0;
      while (p < W) {
        while (p < W && zero(p)) ++p;
        if (p >= W) break;
        int a = p, last = p;
        while (p < W) {
          if (!zero(p)) { last = p; ++p; continue; }
          int zs = p;
          while (p < W && zero(p)) ++p;
          if (p - zs >= 2 || p >= W) break;
        }
        f.m8_seg.push_back(lo + a);
        f.m8_seg.push_back(last - a + 1);
        f.m8_seg.push_back((int)f.m8_w64.size());
        f.m8_seg.push_back(0);
        for (int c = a; c <= last; ++c)
          for (int q = 0; q < G; ++q) f.m8_w64.push_back(dense[(size_t)c * G + q]);
      }
    }
  f.m8_off[(size_t)f.n_tables * ng] = (int)(f.m8_seg.size() / 4);
}

// Debug statistic: density nnz / (G * MSEG columns) of groups of G rows (split at zero runs >= 2).
static double mseg_density(const BandFamily& f, int G) {
  double nnz = 0, cols = 0;
  std::vector<char> any;
  for (int m = 0; m < f.n_tables; ++m)
    for (int g0 = 0; g0 < f.n_rows; g0 += G) {
      int lo = 1 << 30, hi = -1;
      for (int r = g0; r < std::min(f.n_rows, g0 + G); ++r) {
        size_t idx = (size_t)m * f.n_rows + r;
        if (!f.len[idx]) continue;
        lo = std::min(lo, (int)f.start[idx]);
        hi = std::max(hi, (int)(f.start[idx] + f.len[idx]));
      }
      if (hi < 0) continue;
      any.assign(hi - lo, 0);
      for (int r = g0; r < std::min(f.n_rows, g0 + G); ++r) {
        size_t idx = (size_t)m * f.n_rows + r;
        for (int e = 0; e < f.len[idx]; ++e)
          if (f.w64[idx * f.taps + e] != 0.0) { any[f.start[idx] + e - lo] = 1; nnz += 1; }
      }
      int p = 0, W = hi - lo;
      while (p < W) {
        while (p < W && !any[p]) ++p;
        if (p >= W) break;
        int a = p, last = p;
        while (p < W) {
          if (any[p]) { last = p; ++p; continue; }
          int zs = p;
          while (p < W && !any[p]) ++p;
          if (p - zs >= 2 || p >= W) break;
        }
        cols += last - a + 1;
      }
    }
  return nnz / (G * cols);
}

// Slice-interleaved forms of a per-slice family f (n_tables = nz, rows r, sources j):
//  rows_by_slice: one table, row (r, n) at r*nz + n = table n's row r (same sources).  Groups of 4 rows
//                 are then 4 neighbouring slices of one output row, whose bands nearly coincide.
//  cols_by_slice: one table, row r with sources (j, n) at j*nz + n = table n's entry (r, j): the sum over
//                 slices becomes one long band over the interleaved source index.
static void make_rows_by_slice(BandFamily& out, const BandFamily& f) {
  const int nz = f.n_tables;
  family_init(out, 1, f.n_rows * nz, f.n_src);
  FamilyBuilder b(out);
  b.tabs.resize(1);
  b.tabs[0].assign((size_t)f.n_rows * nz, Row());
  for (int r = 0; r < f.n_rows; ++r)
    for (int n = 0; n < nz; ++n) {
      size_t idx = (size_t)n * f.n_rows + r;
      Row& row = b.tabs[0][(size_t)r * nz + n];
      row.lo = f.start[idx];
      row.len = f.len[idx];
      row.w.assign(f.w64.begin() + idx * f.taps, f.w64.begin() + idx * f.taps + f.len[idx]);
    }
  b.finish();
}

static void make_cols_by_slice(BandFamily& out, const BandFamily& f) {
  const int nz = f.n_tables;
  family_init(out, 1, f.n_rows, f.n_src * nz);
  FamilyBuilder b(out);
  b.tabs.resize(1);
  b.tabs[0].assign(f.n_rows, Row());
  for (int r = 0; r < f.n_rows; ++r) {
    int lo = 1 << 30, hi = -1;
    for (int n = 0; n < nz; ++n) {
      size_t idx = (size_t)n * f.n_rows + r;
      if (!f.len[idx]) continue;
      lo = std::min(lo, f.start[idx] * nz + n);
      hi = std::max(hi, (f.start[idx] + f.len[idx] - 1) * nz + n);
    }
    Row& row = b.tabs[0][r];
    if (hi < 0) continue;
    row.lo = lo;
    row.len = hi - lo + 1;
    row.w.assign(row.len, 0.0);
    for (int n = 0; n < nz; ++n) {
      size_t idx = (size_t)n * f.n_rows + r;
      for (int q = 0; q < f.len[idx]; ++q) row.w[(size_t)(f.start[idx] + q) * nz + n - lo] = f.w64[idx * f.taps + q];
    }
  }
  b.finish();
}

static void make_identity(BandFamily& f, int n) {
  family_init(f, 1, n, n);
  FamilyBuilder b(f);
  b.tabs.resize(1);
  b.tabs[0].assign(n, Row());
  for (int r = 0; r < n; ++r) {
    b.tabs[0][r].lo = r;
    b.tabs[0][r].len = 1;
    b.tabs[0][r].w.assign(1, 1.0);
  }
  b.finish();
}

// ------------------------------------------------------------------------------------------
// Rotation (eqn,rot,decomp): closed form, same expression order as DESIGN.md.
struct Decomp {
  double D[3];
  double a_yx, a_yz, a_xy, a_xz, a_zx, a_zy;
};

static lfm_status decompose(const double* T, Decomp& d, std::string& err) {
  double Txx = T[0], Txy = T[1], Txz = T[2], Tyx = T[3], Tyy = T[4], Tyz = T[5], Tzx = T[6], Tzy = T[7], Tzz = T[8];
  double Dy = Tyy;
  if (std::fabs(Dy) < 1e-6) { err = "rotation: D_y ~ 0 (>= 45 deg needs a quarter-turn permutation)"; return LFM_E_DEGENERATE; }
  d.a_yx = Tyx / Dy;
  d.a_yz = Tyz / Dy;
  double Dx = Txx - Txy * d.a_yx;
  if (std::fabs(Dx) < 1e-6) { err = "rotation: D_x ~ 0"; return LFM_E_DEGENERATE; }
  d.a_xy = Txy / Dx;
  d.a_xz = Txz / Dx - d.a_xy * d.a_yz;
  double m_xx = 1.0 + d.a_xy * d.a_yx;
  double m_xz = d.a_xz + d.a_xy * d.a_yz;
  double alpha = Tzx - d.a_yx * Tzy;
  double beta = m_xx * Tzy - d.a_xy * Tzx;
  double Dz = Tzz - alpha * m_xz - beta * d.a_yz;
  if (std::fabs(Dz) < 1e-6) { err = "rotation: D_z ~ 0"; return LFM_E_DEGENERATE; }
  d.a_zx = alpha / Dz;
  d.a_zy = beta / Dz;
  d.D[0] = Dx;
  d.D[1] = Dy;
  d.D[2] = Dz;
  return LFM_OK;
}

// (1/D)(Lambda_D * U_wa * U_wb)(d): exact piecewise polynomial via antiderivatives of Lambda.
static double lam1(double t, double D) {
  if (t <= -D) return 0.0;
  if (t <= 0.0) return 0.5 * (t + D) * (t + D);
  if (t < D) return D * D - 0.5 * (D - t) * (D - t);
  return D * D;
}
static double lam2(double t, double D) {
  if (t <= -D) return 0.0;
  if (t <= 0.0) return (t + D) * (t + D) * (t + D) / 6.0;
  if (t < D) return D * D * t + (D - t) * (D - t) * (D - t) / 6.0;
  return D * D * t;
}
static double shear_weight(double d, double D, double wa, double wb) {
  double tiny = 1e-9 * D;
  double a = std::fabs(wa), b = std::fabs(wb);
  bool ha = a > tiny, hb = b > tiny;
  if (!ha && !hb) return std::max(0.0, D - std::fabs(d)) / D;
  if (ha != hb) {
    double w = ha ? a : b;
    return (lam1(d + 0.5 * w, D) - lam1(d - 0.5 * w, D)) / (w * D);
  }
  double lo = std::min(a, b), hi = std::max(a, b);
  double v = (lam2(d + 0.5 * (lo + hi), D) - lam2(d + 0.5 * (hi - lo), D) - lam2(d - 0.5 * (hi - lo), D) +
              lam2(d - 0.5 * (lo + hi), D)) / (lo * hi * D);
  return std::max(v, 0.0);
}

static void build_shear(ShearPass& sp, int axis, double c1, double c2, const int dims[3], const double vox[3]) {
  sp.axis = axis;
  sp.c1 = c1;
  sp.c2 = c2;
  sp.active = (c1 != 0.0 || c2 != 0.0);
  if (!sp.active) return;
  // axis 0: z-pass, lines (x,y), sigma = c1 x + c2 y, widths c1 dx, c2 dy, D = dz
  // axis 1: x-pass, lines (y,z), sigma = c1 y + c2 z, widths c1 dy, c2 dz, D = dx
  // axis 2: y-pass, lines (x,z), sigma = c1 x + c2 z, widths c1 dx, c2 dz, D = dy
  int a1, a2, al;
  if (axis == 0) { a1 = 0; a2 = 1; al = 2; }
  else if (axis == 1) { a1 = 1; a2 = 2; al = 0; }
  else { a1 = 0; a2 = 2; al = 1; }
  int n1 = dims[a1], n2 = dims[a2];
  double D = vox[al];
  double wa = c1 * vox[a1], wb = c2 * vox[a2];
  double reach = D + 0.5 * (std::fabs(wa) + std::fabs(wb));
  sp.n_lines = n1 * n2;
  int taps = 1;
  std::vector<int> lo_f(sp.n_lines), lo_a(sp.n_lines), hi_f(sp.n_lines), hi_a(sp.n_lines);
  for (int i2 = 0; i2 < n2; ++i2)
    for (int i1 = 0; i1 < n1; ++i1) {
      int line = i1 + n1 * i2;
      double p1 = ((double)i1 - (n1 - 1) * 0.5) * vox[a1];
      double p2 = ((double)i2 - (n2 - 1) * 0.5) * vox[a2];
      double sig = c1 * p1 + c2 * p2;
      for (int dir = 0; dir < 2; ++dir) {
        double s = dir == 0 ? sig : -sig;  // E(a,b)^T = E(-a,-b)
        int lo = (int)std::floor((s - reach) / D) + 1;
        int hi = (int)std::ceil((s + reach) / D) - 1;
        (dir == 0 ? lo_f : lo_a)[line] = lo;
        (dir == 0 ? hi_f : hi_a)[line] = hi;
        taps = std::max(taps, hi - lo + 1);
      }
    }
  int pad = taps <= 4 ? 4 : (taps <= 8 ? 8 : 16);
  sp.taps = pad;
  for (int dir = 0; dir < 2; ++dir) {
    sp.mlo[dir].assign(sp.n_lines, 0);
    sp.w64[dir].assign((size_t)sp.n_lines * pad, 0.0);
    for (int i2 = 0; i2 < n2; ++i2)
      for (int i1 = 0; i1 < n1; ++i1) {
        int line = i1 + n1 * i2;
        double p1 = ((double)i1 - (n1 - 1) * 0.5) * vox[a1];
        double p2 = ((double)i2 - (n2 - 1) * 0.5) * vox[a2];
        double s = c1 * p1 + c2 * p2;
        if (dir) s = -s;
        int lo = (dir == 0 ? lo_f : lo_a)[line];
        int hi = (dir == 0 ? hi_f : hi_a)[line];
        sp.mlo[dir][line] = lo;
        for (int m = lo; m <= hi; ++m) sp.w64[dir][(size_t)line * pad + (m - lo)] = shear_weight(m * D - s, D, wa, wb);
      }
  }
}

// ------------------------------------------------------------------------------------------
// Footprint of table `tab` over output tile t: [lo, lo+width) of source cells (ELL entries).
void ell_footprint(const BandFamily& f, int tab, int tile, int t, int& lo, int& width) {
  size_t per = (size_t)f.ell * f.n_rows;
  int mn = 1 << 30, mxv = -1;
  for (int r = t * tile; r < std::min(f.n_rows, (t + 1) * tile); ++r) {
    int c = f.cnt[(size_t)tab * f.n_rows + r];
    for (int e = 0; e < c; ++e) {
      int j = f.eidx[tab * per + (size_t)e * f.n_rows + r];
      mn = std::min(mn, j);
      mxv = std::max(mxv, j);
    }
  }
  if (mxv < 0) { lo = 0; width = 0; return; }
  lo = mn;
  width = mxv - mn + 1;
}

void fill_sep_geometry(SepOp& op) {
  const BandFamily& fs = *op.fs;
  const BandFamily& ft = *op.ft;
  op.fs_max = 1;
  op.ft_max = 1;
  op.wt_max = 4;
  op.ws_max = 4;
  std::vector<char> seen_s(fs.n_tables, 0), seen_t(ft.n_tables, 0);
  double fma = 0;
  int ntx = (fs.n_rows + op.ts - 1) / op.ts, nty = (ft.n_rows + op.tt - 1) / op.tt;
  std::vector<double> sum_s(fs.n_tables, 0), sum_t(ft.n_tables, 0), used_t(ft.n_tables, 0);
  for (const Term& t : op.terms) {
    if (!seen_s[t.s_tab]) {
      seen_s[t.s_tab] = 1;
      for (int x = 0; x < ntx; ++x) {
        int lo, w, wo, wl;
        g4_tile(fs, t.s_tab, op.ts, x, lo, w, wo, wl);
        op.fs_max = std::max(op.fs_max, w);
        op.ws_max = std::max(op.ws_max, wl);
      }
      for (int r = 0; r < fs.n_rows; ++r) sum_s[t.s_tab] += fs.cnt[(size_t)t.s_tab * fs.n_rows + r];
    }
    if (!seen_t[t.t_tab]) {
      seen_t[t.t_tab] = 1;
      int glo = 1 << 30, ghi = -1;
      for (int y = 0; y < nty; ++y) {
        int lo, w, wo, wl;
        g4_tile(ft, t.t_tab, op.tt, y, lo, w, wo, wl);
        op.ft_max = std::max(op.ft_max, w);
        op.wt_max = std::max(op.wt_max, wl);
        if (w) { glo = std::min(glo, lo); ghi = std::max(ghi, lo + w); }
      }
      used_t[t.t_tab] = ghi > glo ? ghi - glo : 0;
      for (int r = 0; r < ft.n_rows; ++r) sum_t[t.t_tab] += ft.cnt[(size_t)t.t_tab * ft.n_rows + r];
    }
    // algorithmic FMAs (non-zeros only) of the s-then-t evaluation the kernel performs
    fma += used_t[t.t_tab] * sum_s[t.s_tab] + sum_t[t.t_tab] * fs.n_rows;
  }
  op.fma_alg = fma;
  size_t maxt = 0;
  for (size_t b = 0; b + 1 < op.offs.size(); ++b) maxt = std::max(maxt, (size_t)(op.offs[b + 1] - op.offs[b]));
  op.nbuf = maxt > (size_t)op.nb ? 2 : 1;
}

static void sep_init(SepOp& op, const BandFamily* fs, const BandFamily* ft, int n_is, int n_it, int n_out,
                     float out_scale) {
  op.fs = fs;
  op.ft = ft;
  op.n_os = fs->n_rows;
  op.n_ot = ft->n_rows;
  op.n_is = n_is;
  op.n_it = n_it;
  op.n_out = n_out;
  op.out_scale = out_scale;
  op.s_ident = 0;
  op.terms.clear();
  op.offs.assign(1, 0);
}
static void sep_add(SepOp& op, long long off, int s_tab, int t_tab, float scale) {
  op.terms.push_back(Term{off, s_tab, t_tab, scale, 0});
}
static void sep_close_output(SepOp& op) { op.offs.push_back((int32_t)op.terms.size()); }

// Shared memory of one stage of `nb` terms (must match kernels.cu).
size_t sep_smem(const SepOp& op, int nb) {
  // per staged term: source footprint, s weights, s group descriptors, t weights, t group descriptors
  // (must match slot_layout() in kernels.cu); double-buffered when an output has more than nb terms
  auto r4 = [](size_t v) { return (v + 3) / 4 * 4; };
  size_t fsp = (size_t)op.fs_max + 1;
  // staged rows padded by one pass-1 row stride (the kernel reads two rows per step unconditionally)
  size_t gstep = (size_t)op.nt / (op.ts / 4);
  size_t x = (op.s_ident || !op.stage) ? 0 : r4(((size_t)op.ft_max + gstep) * fsp);
  size_t per = x + r4(op.ws_max) + 2 * (size_t)op.ts + r4(op.wt_max) + 2 * (size_t)op.tt;
  size_t urows = (size_t)op.ft_max + gstep;  // U rows padded likewise
  size_t maxt = 0;
  for (size_t b = 0; b + 1 < op.offs.size(); ++b) maxt = std::max(maxt, (size_t)(op.offs[b + 1] - op.offs[b]));
  size_t nbuf = maxt > (size_t)nb ? 2 : 1;
  const bool u_tile = !(op.s_ident && !op.stage);   // identity s read from global: no U tile
  return (nbuf * per * nb + (u_tile ? nbuf * (size_t)nb * urows * op.ts : 0)) * 4;
}
// Estimated time of an op for a tile choice: L2->SM traffic of the staged footprints and the FMA issue
// slots of both passes, with a crude occupancy factor (a sampled cost model).
static double sep_cost(const SepOp& op, int nt, size_t smem) {
  const BandFamily& fs = *op.fs;
  const BandFamily& ft = *op.ft;
  size_t nterms = op.terms.size();
  size_t step = std::max<size_t>(1, nterms / 64);
  double bytes = 0, slots = 0;
  int ntx = (fs.n_rows + op.ts - 1) / op.ts, nty = (ft.n_rows + op.tt - 1) / op.tt;
  for (size_t e = 0; e < nterms; e += step) {
    const Term& t = op.terms[e];
    std::vector<int> flo(ntx), fw(ntx), fwl(ntx);
    for (int x = 0; x < ntx; ++x) {
      int wo;
      g4_tile(fs, t.s_tab, op.ts, x, flo[x], fw[x], wo, fwl[x]);
    }
    for (int y = 0; y < nty; ++y) {
      int lo, w, wo, wl;
      g4_tile(ft, t.t_tab, op.tt, y, lo, w, wo, wl);
      if (!w) continue;
      for (int x = 0; x < ntx; ++x) {
        if (!fw[x]) continue;
        if (op.s_ident) {
          // staged: U tile; unstaged: pass 2 streams the rows from L1/L2 (~2x the L2 traffic of one staging)
          bytes += 4.0 * (double)w * op.ts * (op.stage ? 1.0 : 6.0) + 4.0 * wl;
          slots += (double)wl * op.ts;
        } else {
          // unstaged pass 1 gathers scalar loads from L1/L2: latency-bound, counted 4x
          // unstaged: gathered rows are shared through L1 by the TS/4 column groups of the CTA
          bytes += 4.0 * ((op.stage ? (double)w * fw[x] : 2.0 * w * fwl[x] / 4.0 * (32.0 / op.ts)) + fwl[x] + wl);
          slots += 1.3 * (double)w * fwl[x] * (op.stage ? 1.0 : 1.5) + (double)wl * op.ts;  // pass 1 + pass 2
        }
      }
    }
  }
  double scale = (double)nterms / ((nterms + step - 1) / step);
  int ctas = (int)std::max<size_t>(1, (228 * 1024) / (smem + 1024));
  ctas = std::min(ctas, 2048 / nt);
  ctas = std::min(ctas, 65536 / (nt * 96));          // ~96 registers per thread
  double occ = std::min(1.0, ctas * nt / 1024.0);     // latency-bound below ~32 warps per SM (measured)
  return scale * (bytes / 6e12 + slots / (30e12 * occ));
}

bool sep_choose_tile(SepOp& op) {
  const int cand[][3] = {{128, 64, 256}, {128, 32, 256}, {64, 64, 128}, {64, 32, 128}, {32, 32, 64}};
  double best = 1e300;
  int bts = 0, btt = 0, bst = 0, bnb = 0, bnt = 0;
  for (auto& c : cand) {
    for (int stage : {1, 0}) {
      op.ts = c[0];
      op.tt = c[1];
      op.nt = c[2];
      op.stage = stage;
      fill_sep_geometry(op);
      for (int nb : {4, 2, 1}) {
        if (nb > 1 && op.terms.size() < (size_t)op.n_out * 2) continue;  // single-term outputs: nb = 1
        size_t smem = sep_smem(op, nb);
        if (smem > (size_t)210 * 1024) continue;
        double cost = sep_cost(op, c[2], smem) * (nb == 1 && op.terms.size() >= (size_t)op.n_out * 2 ? 1.1 : 1.0);
        if (cost < best) { best = cost; bts = c[0]; btt = c[1]; bst = stage; bnb = nb; bnt = c[2]; }
      }
    }
  }
  if (!bts) return false;
  op.ts = bts;
  op.tt = btt;
  op.stage = bst;
  op.nb = bnb;
  op.nt = bnt;
  fill_sep_geometry(op);
  return true;
}

// ------------------------------------------------------------------------------------------
// Collapsed composite of one axis over the views k_axis with kmask[k] != 0, per slice n (NEXT-1):
//   C_n = scale * sum_k S_k B_{k,n} (plenoptic, S_k the masked lenslet stage) or scale * sum_k B_{k,n} (single),
// built in fp64 from the per-view band tables; cf = C_n (rows: detector cells), ca = C_n^T (rows: voxel cells).
// The band of a composite row is the union of the S1 bands its non-zero S3 entries reach (structural zeros
// between two lenslets' cells are skipped).
static void build_composite(const CameraPlan& cp, int ax, const std::vector<char>& kmask, double scale, int nz,
                            int nrow, int nv, bool plen, BandFamily& cf, BandFamily& ca, int tau) {
  const BandFamily& f1 = cp.s1f[ax];
  const int Kax = (int)kmask.size();
  const int keep_f = cf.want_mseg, keep_a = ca.want_mseg;
  family_init(cf, nz, nrow, nv);
  family_init(ca, nz, nv, nrow);
  cf.want_mseg = keep_f;
  ca.want_mseg = keep_a;
  FamilyBuilder bf(cf), ba(ca);
  bf.tabs.resize(nz);
  ba.tabs.resize(nz);
  std::vector<double> accv(nv);
  std::vector<char> touched(nv);
  for (int n = 0; n < nz; ++n) {
    auto& rows = bf.tabs[n];
    rows.assign(nrow, Row());
    std::vector<std::vector<std::pair<int, double>>> cols(nv);  // transpose
    for (int i = 0; i < nrow; ++i) {
      std::fill(accv.begin(), accv.end(), 0.0);
      std::fill(touched.begin(), touched.end(), 0);
      int vlo = 1 << 30, vhi = -1;
      for (int k = 0; k < Kax; ++k) {
        if (!kmask[k]) continue;
        auto add_s1 = [&](int j, double w3) {
          size_t idx = (size_t)(k * nz + n) * f1.n_rows + j;
          for (int q = 0; q < f1.len[idx]; ++q) {
            int v = f1.start[idx] + q;
            accv[v] += w3 * f1.w64[idx * f1.taps + q];
            touched[v] = 1;
            vlo = std::min(vlo, v);
            vhi = std::max(vhi, v);
          }
        };
        if (plen) {
          const BandFamily& f3 = cp.s3f[ax];
          size_t i3 = (size_t)(k * cp.n_terms + tau) * f3.n_rows + i;
          for (int q = 0; q < f3.len[i3]; ++q) {
            double w3 = f3.w64[i3 * f3.taps + q];
            if (w3 == 0.0) continue;  // gap between two lenslets' cells (structural zero)
            add_s1(f3.start[i3] + q, w3);
          }
        } else {
          add_s1(i, 1.0);
        }
      }
      if (vhi < 0) continue;
      Row& r = rows[i];
      r.lo = vlo;
      r.len = vhi - vlo + 1;
      r.w.assign(r.len, 0.0);
      for (int v = vlo; v <= vhi; ++v) {
        r.w[v - vlo] = scale * accv[v];
        if (touched[v]) cols[v].push_back({i, scale * accv[v]});
      }
    }
    auto& arows = ba.tabs[n];
    arows.assign(nv, Row());
    for (int v = 0; v < nv; ++v) {
      if (cols[v].empty()) continue;
      Row& r = arows[v];
      r.lo = cols[v].front().first;
      r.len = cols[v].back().first - r.lo + 1;
      r.w.assign(r.len, 0.0);
      for (auto& e : cols[v]) r.w[e.first - r.lo] = e.second;
    }
  }
  bf.finish();
  ba.finish();
}

lfm_status build_camera(const lfm_volume& vol, const lfm_camera& cam, int n_subsets, CameraPlan& cp,
                        std::string& err) {
  cp.cam = cam;
  lfm_info& info = cp.info;
  std::memset(&info, 0, sizeof(info));
  if (vol.nx <= 0 || vol.ny <= 0 || vol.nz <= 0 || !(vol.dx > 0) || !(vol.dy > 0) || !(vol.dz > 0)) {
    err = "invalid volume";
    return LFM_E_INVALID;
  }
  if (cam.k_s <= 0 || cam.k_t <= 0 || cam.n_s <= 0 || cam.n_t <= 0 || !(cam.px_s > 0) || !(cam.px_t > 0) ||
      !(cam.ap_s > 0) || !(cam.ap_t > 0) || (cam.basis != LFM_PILLBOX && cam.basis != LFM_DIRAC)) {
    err = "invalid camera parameters";
    return LFM_E_INVALID;
  }
  if (cam.f_main == 0.0) { err = "zero main-lens focal length"; return LFM_E_SINGULAR; }
  const bool plen = cam.type == LFM_PLENOPTIC;
  if (plen) {
    if (cam.nl_s <= 0 || cam.nl_t <= 0 || cam.n_a <= 0 || !(cam.fill > 0) || cam.fill > 1.0) {
      err = "invalid plenoptic parameters (nl, n_a > 0, 0 < fill <= 1)";
      return LFM_E_INVALID;
    }
    if (cam.f_mu == 0.0) { err = "zero lenslet focal length"; return LFM_E_SINGULAR; }
  } else if (cam.type != LFM_SINGLE) {
    err = "unknown camera type";
    return LFM_E_INVALID;
  }
  // reading R7: Theta = P Theta' with P the cube rotation of largest trace(P^T Theta) (identity first, then
  // permutations in lexicographic order x sign patterns (+,+,+), (+,+,-), ...; ties keep the earlier one)
  const int dims[3] = {vol.nx, vol.ny, vol.nz};
  const double vox[3] = {vol.dx, vol.dy, vol.dz};
  double Tres[9];
  {
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    double best = -1e300;
    int bp[3] = {0, 1, 2}, bs[3] = {1, 1, 1};
    auto consider = [&](const int* pm, const int* sg) {
      double tr = 0;  // trace(P^T T) = sum_r s_r T[r][pm[r]]
      for (int r = 0; r < 3; ++r) tr += sg[r] * cam.R[3 * r + pm[r]];
      if (tr > best + 1e-12) {
        best = tr;
        for (int r = 0; r < 3; ++r) { bp[r] = pm[r]; bs[r] = sg[r]; }
      }
    };
    const int id[3] = {0, 1, 2}, one[3] = {1, 1, 1};
    consider(id, one);
    for (int q = 0; q < 6; ++q)
      for (int m = 0; m < 8; ++m) {
        const int sg[3] = {(m & 4) ? -1 : 1, (m & 2) ? -1 : 1, (m & 1) ? -1 : 1};
        // det of a signed permutation = sign(perm) * s0 s1 s2
        const int par = (q == 0 || q == 3 || q == 4) ? 1 : -1;
        if (par * sg[0] * sg[1] * sg[2] != 1) continue;
        if (q == 0 && m == 0) continue;  // identity already considered
        consider(perms[q], sg);
      }
    // Tres = P^T T: row a of P^T T = sum_r P[r][a] T[r][.] -> P[r][bp[r]] = bs[r]
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) Tres[3 * bp[r] + c] = bs[r] * cam.R[3 * r + c];
    cp.has_perm = !(bp[0] == 0 && bp[1] == 1 && bp[2] == 2 && bs[0] == 1 && bs[1] == 1 && bs[2] == 1);
    for (int k = 0; k < 9; ++k) info.rot_perm[k] = 0;
    for (int r = 0; r < 3; ++r) info.rot_perm[3 * r + bp[r]] = bs[r];
    if (cp.has_perm) {
      for (int b = 0; b < 3; ++b) {
        const int a = bp[b];
        if (dims[a] != dims[b] || std::fabs(vox[a] - vox[b]) > 1e-12 * vox[b]) {
          err = "pose needs a quarter-turn relabelling, which needs equal dims and voxel sizes on the permuted axes";
          return LFM_E_DEGENERATE;
        }
        // forward x_P(q) = x(P q): source axis of output axis b is bp[b] with sign bs[b];
        // adjoint (P^T): output axis bp[b] reads source axis b with the same sign
        cp.perm_axis[0][b] = bp[b];
        cp.perm_sign[0][b] = bs[b];
        cp.perm_axis[1][bp[b]] = b;
        cp.perm_sign[1][bp[b]] = bs[b];
      }
    }
  }
  Decomp dec;
  lfm_status st = decompose(Tres, dec, err);
  if (st != LFM_OK) return st;
  double vox_r[3] = {vox[0] / dec.D[0], vox[1] / dec.D[1], vox[2] / dec.D[2]};
  const int nx = vol.nx, ny = vol.ny, nz = vol.nz;
  info.type = cam.type;
  info.basis = cam.basis;
  info.nx = nx; info.ny = ny; info.nz = nz;
  info.n_vox = (long long)nx * ny * nz;
  info.n_s = cam.n_s; info.n_t = cam.n_t;
  info.n_pix = (long long)cam.n_s * cam.n_t;
  info.k_s = cam.k_s; info.k_t = cam.k_t;
  info.n_views = cam.k_s * cam.k_t;
  for (int a = 0; a < 3; ++a) { info.vox_r[a] = vox_r[a]; info.rot_D[a] = dec.D[a]; }
  info.shear[0] = dec.a_zx; info.shear[1] = dec.a_zy; info.shear[2] = dec.a_xy;
  info.shear[3] = dec.a_xz; info.shear[4] = dec.a_yx; info.shear[5] = dec.a_yz;
  info.plane_array = plen ? nz : -1;
  info.plane_detector = nz + 1;

  // rotation passes in application order z, x, y
  build_shear(cp.rot[0], 0, dec.a_zx, dec.a_zy, dims, vox_r);
  build_shear(cp.rot[1], 1, dec.a_xy, dec.a_xz, dims, vox_r);
  build_shear(cp.rot[2], 2, dec.a_yx, dec.a_yz, dims, vox_r);
  info.rot_passes = (cp.rot[0].active ? 1 : 0) | (cp.rot[1].active ? 2 : 0) | (cp.rot[2].active ? 4 : 0) |
                    (cp.has_perm ? 8 : 0);

  // planes per axis
  const int K[2] = {cam.k_s, cam.k_t};
  const double d0[2] = {cam.ap_s / cam.k_s, cam.ap_t / cam.k_t};
  const int nsrc[2] = {nx, ny};
  const int ndet[2] = {cam.n_s, cam.n_t};
  const double pdet[2] = {cam.px_s, cam.px_t};
  const int nl[2] = {cam.nl_s, cam.nl_t};
  const double dz = vox_r[2];
  std::vector<double> zs(nz);
  for (int n = 0; n < nz; ++n) zs[n] = cam.d_scene + ((double)n - (nz - 1) * 0.5) * dz;

  Plane dst[2];
  double V_dst[2], V_mu[2] = {0, 0};
  double pitch[2] = {0, 0};
  for (int ax = 0; ax < 2; ++ax) {
    if (plen) {
      pitch[ax] = ndet[ax] * pdet[ax] / nl[ax];
      dst[ax] = Plane{nl[ax] * cam.n_a, pitch[ax] / cam.n_a, translate(-cam.d_mu_m), 0.0};
    } else {
      dst[ax] = Plane{ndet[ax], pdet[ax], translate(-cam.d_det), 0.0};
    }
    V_dst[ax] = basis_volume(dst[ax], d0[ax]);
  }
  // ---- lenslet stage (plenoptic) as a sum of T separable terms (readings Z9/Z10, R12, R13):
  //   S_k = sum_mu c3 B^{d mu}_k M_mu = sum_tau c3 S^tau_{k,s} (x) S^tau_{k,t},
  // term tau = per axis a list of items (lenslet plane along the axis, open array cells [lo, hi] along it).
  // Rectangular grid + square apertures: one term, per axis every lenslet with its open interval.  Hexagonal layout
  // (odd lenslet rows shifted by pitch_s / 2, one lenslet fewer) and/or circular apertures (cells whose centres lie
  // strictly inside the disk of diameter fill * pitch_s): each (lenslet row j, array row j_t) pair contributes the
  // row's open s-cells of row j's lenslets; pairs with the same parity of j and the same s-cells form one term
  // (its t items: the rows j_t, each through its own lenslet row's plane).
  struct Item { int plane, lo, hi; };
  std::vector<Plane> lplanes[2];
  std::vector<std::vector<Item>> terms[2];
  int T = 1;
  if (plen) {
    if ((cam.lens_layout != 0 && cam.lens_layout != 1) || (cam.aperture != 0 && cam.aperture != 1)) {
      err = "lens_layout and aperture must be 0 or 1";
      return LFM_E_INVALID;
    }
    if (cam.lens_layout == 1 && cam.nl_s < 2) { err = "a hexagonal lenslet layout needs nl_s >= 2"; return LFM_E_INVALID; }
    std::vector<double> pl_c[2];  // centre of each plane along each axis
    auto plane_of = [&](int ax, double c, int& idx) -> lfm_status {
      for (size_t q = 0; q < pl_c[ax].size(); ++q)
        if (pl_c[ax][q] == c) { idx = (int)q; return LFM_OK; }
      Affine inv;
      if (!invert(lens(cam.f_mu, c), inv)) { err = "singular lenslet block"; return LFM_E_SINGULAR; }
      Affine X0 = compose(translate(-cam.d_mu_m), compose(inv, translate(-cam.d_d_mu)));
      lplanes[ax].push_back(Plane{ndet[ax], pdet[ax], X0, 0.0});
      pl_c[ax].push_back(c);
      idx = (int)pl_c[ax].size() - 1;
      return LFM_OK;
    };
    const bool sep_geom = cam.lens_layout == 0 && cam.aperture == 0;
    if (sep_geom) {
      for (int ax = 0; ax < 2; ++ax) {
        terms[ax].assign(1, {});
        for (int mu = 0; mu < nl[ax]; ++mu) {
          double c_mu = ((double)mu - (nl[ax] - 1) * 0.5) * pitch[ax];
          int pi;
          if ((st = plane_of(ax, c_mu, pi)) != LFM_OK) return st;
          double half = 0.5 * cam.fill * pitch[ax];
          int lo = 1 << 30, hi = -1;
          for (int j = 0; j < dst[ax].n; ++j) {
            double c = centre(dst[ax], j);
            if (c >= c_mu - half && c < c_mu + half) { lo = std::min(lo, j); hi = std::max(hi, j); }
          }
          if (hi >= lo) terms[ax][0].push_back({pi, lo, hi});
        }
      }
    } else {
      const int nas = dst[0].n, nat = dst[1].n;
      std::vector<int> owners((size_t)nas * nat, 0);
      std::map<std::vector<int>, int> key_to_term;
      for (int j = 0; j < nl[1]; ++j) {
        const bool odd = cam.lens_layout == 1 && (j & 1);
        const double c_t = ((double)j - (nl[1] - 1) * 0.5) * pitch[1];
        int pt;
        if ((st = plane_of(1, c_t, pt)) != LFM_OK) return st;
        // per array row: the open s-interval of each lenslet of this lenslet row
        std::vector<std::vector<int>> row_key(nat);   // [parity, plane, lo, hi, plane, lo, hi, ...]
        for (int i = 0; i < nl[0] - (odd ? 1 : 0); ++i) {
          const double c_s = ((double)i - (nl[0] - 1) * 0.5 + (odd ? 0.5 : 0.0)) * pitch[0];
          int ps;
          if ((st = plane_of(0, c_s, ps)) != LFM_OK) return st;
          for (int jt = 0; jt < nat; ++jt) {
            const double tt = centre(dst[1], jt);
            int lo = 1 << 30, hi = -1;
            for (int js = 0; js < nas; ++js) {
              const double ss = centre(dst[0], js);
              bool open;
              if (cam.aperture == 1) {
                const double r = 0.5 * cam.fill * pitch[0];
                open = (ss - c_s) * (ss - c_s) + (tt - c_t) * (tt - c_t) < r * r;
              } else {
                const double hs = 0.5 * cam.fill * pitch[0], ht = 0.5 * cam.fill * pitch[1];
                open = ss >= c_s - hs && ss < c_s + hs && tt >= c_t - ht && tt < c_t + ht;
              }
              if (open) {
                lo = std::min(lo, js);
                hi = std::max(hi, js);
                ++owners[(size_t)jt * nas + js];
              }
            }
            if (hi < 0) continue;
            if (row_key[jt].empty()) row_key[jt].push_back(odd ? 1 : 0);
            row_key[jt].insert(row_key[jt].end(), {ps, lo, hi});
          }
        }
        for (int jt = 0; jt < nat; ++jt) {
          if (row_key[jt].empty()) continue;
          auto it = key_to_term.find(row_key[jt]);
          int tau;
          if (it == key_to_term.end()) {
            tau = (int)terms[0].size();
            key_to_term[row_key[jt]] = tau;
            std::vector<Item> sitems;
            for (size_t q = 1; q + 2 < row_key[jt].size(); q += 3)
              sitems.push_back({row_key[jt][q], row_key[jt][q + 1], row_key[jt][q + 2]});
            terms[0].push_back(sitems);
            terms[1].push_back({});
          } else {
            tau = it->second;
          }
          terms[1][tau].push_back({pt, jt, jt});
        }
      }
      for (int v : owners)
        if (v > 1) { err = "lenslet apertures overlap on the array grid (reduce fill)"; return LFM_E_INVALID; }
      for (auto& tl : terms[1]) {   // within a term every array row has one lenslet row
        std::sort(tl.begin(), tl.end(), [](const Item& a, const Item& b) { return a.lo < b.lo; });
        for (size_t q = 1; q < tl.size(); ++q)
          if (tl[q].lo == tl[q - 1].lo) { err = "lenslet rows share an array row within one term"; return LFM_E_INVALID; }
      }
      if (terms[0].empty()) { terms[0].assign(1, {}); terms[1].assign(1, {}); }
    }
    T = (int)terms[0].size();
    for (int ax = 0; ax < 2; ++ax) V_mu[ax] = basis_volume(lplanes[ax][0], d0[ax]);
  }
  cp.n_terms = T;
  info.s3_terms = T;
  info.n_as = plen ? dst[0].n : 0;
  info.n_at = plen ? dst[1].n : 0;
  const double Vdst = V_dst[0] * V_dst[1];
  const double Vmu = V_mu[0] * V_mu[1];
  // scalars: c1 = dz/V^a (plenoptic) or dz*sqrt(V^d)/V^d (single); c3 = sqrt(V^mu)/V^mu (Z7)
  const double c1 = plen ? dz / Vdst : dz * std::sqrt(Vdst) / Vdst;
  const double c3 = plen ? std::sqrt(Vmu) / Vmu : 1.0;
  cp.scal[0] = c1; cp.scal[1] = c3; cp.scal[2] = Vdst; cp.scal[3] = Vmu; cp.scal[4] = dz;
  cp.scal[5] = d0[0]; cp.scal[6] = d0[1]; cp.scal[7] = plen ? 1.0 : 0.0;

  // ---- S1 families: slice n -> dst (fwd) and dst -> slice n (adj), per axis, table = k*nz + n
  for (int ax = 0; ax < 2; ++ax) {
    family_init(cp.s1f[ax], K[ax] * nz, dst[ax].n, nsrc[ax]);
    family_init(cp.s1a[ax], K[ax] * nz, nsrc[ax], dst[ax].n);
    FamilyBuilder bf(cp.s1f[ax]), ba(cp.s1a[ax]);
    bf.tabs.resize(K[ax] * nz);
    ba.tabs.resize(K[ax] * nz);
    for (int k = 0; k < K[ax]; ++k) {
      double sk = ((double)k - (K[ax] - 1) * 0.5) * d0[ax];
      for (int n = 0; n < nz; ++n) {
        Plane q{nsrc[ax], vox_r[ax], compose(lens(cam.f_main, 0.0), translate(zs[n])), 0.0};
        st = transport_rows(q, dst[ax], sk, d0[ax], cam.basis, bf.tabs[k * nz + n], err);
        if (st != LFM_OK) return st;
        st = transport_rows(dst[ax], q, sk, d0[ax], cam.basis, ba.tabs[k * nz + n], err);
        if (st != LFM_OK) return st;
      }
    }
    bf.finish();
    ba.finish();
  }
  // ---- S3 families (plenoptic), table = k*T + tau: array -> detector through the term's items, masked (fwd),
  //      and detector -> array through the item owning each cell (adj)
  if (plen) {
    for (int ax = 0; ax < 2; ++ax) {
      family_init(cp.s3f[ax], K[ax] * T, ndet[ax], dst[ax].n);
      family_init(cp.s3a[ax], K[ax] * T, dst[ax].n, ndet[ax]);
      FamilyBuilder bf(cp.s3f[ax]), ba(cp.s3a[ax]);
      bf.tabs.resize(K[ax] * T);
      ba.tabs.resize(K[ax] * T);
      for (int k = 0; k < K[ax]; ++k) {
        double sk = ((double)k - (K[ax] - 1) * 0.5) * d0[ax];
        for (int tau = 0; tau < T; ++tau) {
          const std::vector<Item>& items = terms[ax][tau];
          // forward: union over items of band_mu(i) cap the item's open cells
          std::vector<int> lo(ndet[ax], 1 << 30), hi(ndet[ax], -1);
          std::vector<std::vector<std::pair<int, double>>> acc(ndet[ax]);
          for (const Item& it : items) {
            Kernel1D kk;
            st = make_kernel(dst[ax], lplanes[ax][it.plane], sk, d0[ax], cam.basis, kk, err);
            if (st != LFM_OK) return st;
            for (int i = 0; i < ndet[ax]; ++i) {
              double c;
              int blo, bhi;
              row_band(dst[ax], lplanes[ax][it.plane], kk, i, c, blo, bhi);
              blo = std::max(blo, it.lo);
              bhi = std::min(bhi, it.hi);
              if (bhi < blo) continue;
              for (int j = blo; j <= bhi; ++j) acc[i].push_back({j, entry(dst[ax], kk, c, j)});
              lo[i] = std::min(lo[i], blo);
              hi[i] = std::max(hi[i], bhi);
            }
          }
          auto& rows = bf.tabs[k * T + tau];
          rows.assign(ndet[ax], Row());
          for (int i = 0; i < ndet[ax]; ++i) {
            if (hi[i] < 0) continue;
            rows[i].lo = lo[i];
            rows[i].len = hi[i] - lo[i] + 1;
            rows[i].w.assign(rows[i].len, 0.0);
            for (auto& e : acc[i]) rows[i].w[e.first - lo[i]] += e.second;
          }
          // adjoint: row j (array cell) = B^{a mu(j)}[j, :] (transport detector(mu) -> array)
          auto& arows = ba.tabs[k * T + tau];
          arows.assign(dst[ax].n, Row());
          for (const Item& it : items) {
            Kernel1D kk;
            st = make_kernel(lplanes[ax][it.plane], dst[ax], sk, d0[ax], cam.basis, kk, err);
            if (st != LFM_OK) return st;
            for (int j = it.lo; j <= it.hi; ++j) {
              double c;
              int blo, bhi;
              row_band(lplanes[ax][it.plane], dst[ax], kk, j, c, blo, bhi);
              if (bhi < blo) continue;
              Row& r = arows[j];
              r.lo = blo;
              r.len = bhi - blo + 1;
              r.w.resize(r.len);
              for (int i = blo; i <= bhi; ++i) r.w[i - blo] = entry(lplanes[ax][it.plane], kk, c, i);
            }
          }
        }
      }
      bf.finish();
      ba.finish();
    }
  }
  // ---- collapsed composite per slice and term: C^tau_n = sum_k S^tau_k B_{k,n} (plenoptic) or sum_k B_{k,n} (single);
  //      term 0 in the camera's own families, terms >= 1 in cp.comps
  cp.comps.assign(T - 1, Component());
  for (int ax = 0; ax < 2; ++ax) {
    // s-axis composites also serve as t families of the transposed two-pass path (MSEG segments)
    cp.cf[ax].want_mseg = cp.ca[ax].want_mseg = ax == 0;
    build_composite(cp, ax, std::vector<char>(K[ax], 1), 1.0, nz, ndet[ax], nsrc[ax], plen, cp.cf[ax], cp.ca[ax], 0);
    for (int tau = 1; tau < T; ++tau)
      build_composite(cp, ax, std::vector<char>(K[ax], 1), 1.0, nz, ndet[ax], nsrc[ax], plen, cp.comps[tau - 1].cf[ax],
                      cp.comps[tau - 1].ca[ax], tau);
  }
  info.taps_s1 = std::max(cp.s1f[0].ell, cp.s1f[1].gmax);
  info.taps_s3 = plen ? std::max(cp.s3f[0].ell, cp.s3f[1].gmax) : 0;
  info.taps_c = std::max(cp.cf[0].ell, cp.cf[1].gmax);

  // ---- term lists ----
  const int Kv = K[0] * K[1];
  const long long nslice = (long long)nx * ny;
  const long long nfield = plen ? (long long)dst[0].n * dst[1].n : 0;
  const long long npix = (long long)ndet[0] * ndet[1];
  auto tab = [&](int k_axis, int n) { return k_axis * nz + n; };
  if (plen) {
    // forward S1: output k (array field of view k) = c1 * sum_n B^{a q_n}_k x^r_n
    sep_init(cp.fwd_s1, &cp.s1f[0], &cp.s1f[1], nx, ny, Kv, (float)c1);
    for (int kt = 0; kt < K[1]; ++kt)
      for (int ks = 0; ks < K[0]; ++ks) {
        for (int n = 0; n < nz; ++n) sep_add(cp.fwd_s1, n * nslice, tab(ks, n), tab(kt, n), 1.f);
        sep_close_output(cp.fwd_s1);
      }
    // forward S3: y = c3 * sum_k sum_tau (S^tau_ks (x) S^tau_kt) a_k
    sep_init(cp.fwd_s3, &cp.s3f[0], &cp.s3f[1], dst[0].n, dst[1].n, 1, (float)c3);
    for (int kt = 0; kt < K[1]; ++kt)
      for (int ks = 0; ks < K[0]; ++ks)
        for (int tau = 0; tau < T; ++tau)
          sep_add(cp.fwd_s3, (long long)(kt * K[0] + ks) * nfield, ks * T + tau, kt * T + tau, 1.f);
    sep_close_output(cp.fwd_s3);
    // adjoint S3: field k = c3 * S_k^T r  (evaluated with the detector -> array transport)
    sep_init(cp.adj_s3, &cp.s3a[0], &cp.s3a[1], ndet[0], ndet[1], Kv, (float)c3);
    for (int kt = 0; kt < K[1]; ++kt)
      for (int ks = 0; ks < K[0]; ++ks) {
        for (int tau = 0; tau < T; ++tau) sep_add(cp.adj_s3, 0, ks * T + tau, kt * T + tau, 1.f);
        sep_close_output(cp.adj_s3);
      }
    // adjoint S1: slice n = c1 * sum_k B^{q_n a}_k field_k
    sep_init(cp.adj_s1, &cp.s1a[0], &cp.s1a[1], dst[0].n, dst[1].n, nz, (float)c1);
    for (int n = 0; n < nz; ++n) {
      for (int kt = 0; kt < K[1]; ++kt)
        for (int ks = 0; ks < K[0]; ++ks)
          sep_add(cp.adj_s1, (long long)(kt * K[0] + ks) * nfield, tab(ks, n), tab(kt, n), 1.f);
      sep_close_output(cp.adj_s1);
    }
  } else {
    sep_init(cp.fwd_s1, &cp.s1f[0], &cp.s1f[1], nx, ny, 1, (float)c1);
    for (int kt = 0; kt < K[1]; ++kt)
      for (int ks = 0; ks < K[0]; ++ks)
        for (int n = 0; n < nz; ++n) sep_add(cp.fwd_s1, n * nslice, tab(ks, n), tab(kt, n), 1.f);
    sep_close_output(cp.fwd_s1);
    sep_init(cp.adj_s1, &cp.s1a[0], &cp.s1a[1], ndet[0], ndet[1], nz, (float)c1);
    for (int n = 0; n < nz; ++n) {
      for (int kt = 0; kt < K[1]; ++kt)
        for (int ks = 0; ks < K[0]; ++ks) sep_add(cp.adj_s1, 0, tab(ks, n), tab(kt, n), 1.f);
      sep_close_output(cp.adj_s1);
    }
  }
  // view-subset ops (sec,subset): subset m = views k = kt*K_s + ks with k mod M == m, compact field slots,
  // the K/|S| factor of eqn,subset folded into the final op's scale
  cp.subs.clear();
  if (n_subsets > 1) {
    if (n_subsets > Kv) { err = "n_subsets exceeds the number of views"; return LFM_E_INVALID; }
    cp.subs.resize(n_subsets);
    for (int m = 0; m < n_subsets; ++m) {
      ViewOps& vo = cp.subs[m];
      std::vector<int> S;
      for (int k = m; k < Kv; k += n_subsets) S.push_back(k);
      vo.n_views = (int)S.size();
      const double sc = (double)Kv / S.size();
      // tensor-product subset with every k_t: the s composite over S_s, scaled by K/|S|, on the collapsed path
      {
        std::vector<char> in_s(K[0], 0), in_t(K[1], 0);
        for (int k : S) { in_s[k % K[0]] = 1; in_t[k / K[0]] = 1; }
        int ns = 0, nt_ = 0;
        for (char v : in_s) ns += v;
        for (char v : in_t) nt_ += v;
        if (nt_ == K[1] && ns * nt_ == (int)S.size() && T == 1 && !std::getenv("LFM_SUBSET_PER_VIEW")) {
          vo.collapsed = 1;
          build_composite(cp, 0, in_s, sc, nz, ndet[0], nsrc[0], plen, vo.cfs, vo.cas, 0);
        }
      }
      if (plen) {
        sep_init(vo.fwd_s1, &cp.s1f[0], &cp.s1f[1], nx, ny, vo.n_views, (float)c1);
        for (int k : S) {
          const int ks = k % K[0], kt = k / K[0];
          for (int n = 0; n < nz; ++n) sep_add(vo.fwd_s1, n * nslice, tab(ks, n), tab(kt, n), 1.f);
          sep_close_output(vo.fwd_s1);
        }
        sep_init(vo.fwd_s3, &cp.s3f[0], &cp.s3f[1], dst[0].n, dst[1].n, 1, (float)(c3 * sc));
        for (size_t j = 0; j < S.size(); ++j)
          for (int tau = 0; tau < T; ++tau)
            sep_add(vo.fwd_s3, (long long)j * nfield, (S[j] % K[0]) * T + tau, (S[j] / K[0]) * T + tau, 1.f);
        sep_close_output(vo.fwd_s3);
        sep_init(vo.adj_s3, &cp.s3a[0], &cp.s3a[1], ndet[0], ndet[1], vo.n_views, (float)c3);
        for (int k : S) {
          for (int tau = 0; tau < T; ++tau) sep_add(vo.adj_s3, 0, (k % K[0]) * T + tau, (k / K[0]) * T + tau, 1.f);
          sep_close_output(vo.adj_s3);
        }
        sep_init(vo.adj_s1, &cp.s1a[0], &cp.s1a[1], dst[0].n, dst[1].n, nz, (float)(c1 * sc));
        for (int n = 0; n < nz; ++n) {
          for (size_t j = 0; j < S.size(); ++j)
            sep_add(vo.adj_s1, (long long)j * nfield, tab(S[j] % K[0], n), tab(S[j] / K[0], n), 1.f);
          sep_close_output(vo.adj_s1);
        }
      } else {
        sep_init(vo.fwd_s1, &cp.s1f[0], &cp.s1f[1], nx, ny, 1, (float)(c1 * sc));
        for (int k : S)
          for (int n = 0; n < nz; ++n) sep_add(vo.fwd_s1, n * nslice, tab(k % K[0], n), tab(k / K[0], n), 1.f);
        sep_close_output(vo.fwd_s1);
        sep_init(vo.adj_s1, &cp.s1a[0], &cp.s1a[1], ndet[0], ndet[1], nz, (float)(c1 * sc));
        for (int n = 0; n < nz; ++n) {
          for (int k : S) sep_add(vo.adj_s1, 0, tab(k % K[0], n), tab(k / K[0], n), 1.f);
          sep_close_output(vo.adj_s1);
        }
      }
    }
  }
  // slice-interleaved t families of the two-pass collapsed path, with their MSEG segment lists
  cp.ca1n.want_mseg = 1;
  make_rows_by_slice(cp.ca1n, cp.ca[1]);
  build_mseg8(cp.ca1n);
  if (nz % 64 == 0 && !std::getenv("LFM_UMMA_ROWS128")) {
    cp.ca1n.u_mode = 1;
    cp.ca1n.u_nz = nz;
  }
  build_umma(cp.ca1n);
  cp.cf1n.want_mseg = 1;
  make_cols_by_slice(cp.cf1n, cp.cf[1]);
  build_mseg8(cp.cf1n);
  build_umma(cp.cf1n);
  if (std::getenv("LFM_DEBUG")) {
    const BandFamily* fs[] = {&cp.ca1n, &cp.cf1n, &cp.ca[1], &cp.cf[1], &cp.ca[0], &cp.cf[0]};
    const char* nm[] = {"ca1 rows-by-slice", "cf1 cols-by-slice", "ca1", "cf1", "ca0", "cf0"};
    for (int i = 0; i < 6; ++i)
      std::fprintf(stderr, "[lfm] %-18s G4 %.3f  MSEG %.3f  (%.2f segs/group, %.1f cols/seg)  gap-free %.3f\n", nm[i],
                   fs[i]->st_nnz / (4 * fs[i]->st_cols_g4), fs[i]->st_nnz / (4 * fs[i]->st_cols_m),
                   fs[i]->st_msegs / ((double)fs[i]->n_tables * fs[i]->n_groups), fs[i]->st_cols_m / fs[i]->st_msegs,
                   fs[i]->st_nnz / (4 * fs[i]->st_cols_nz));
    for (const BandFamily* f : {&cp.ca1n, &cp.cf1n}) {
      double nnz = 0;
      for (int v : f->cnt) nnz += v;
      int bmin = 1 << 30, bmax = 0;
      for (size_t t = 0; t + 1 < f->u_off.size(); ++t) {
        bmin = std::min(bmin, f->u_off[t + 1] - f->u_off[t]);
        bmax = std::max(bmax, f->u_off[t + 1] - f->u_off[t]);
      }
      std::fprintf(stderr, "[lfm] tcgen05 form: %zu blocks of 128x16, density %.3f, %d tiles, blocks per tile %d..%d\n",
                   f->u_k0.size(), nnz / (2048.0 * f->u_k0.size()), (int)f->u_off.size() - 1, bmin, bmax);
      {  // persistent-CTA load balance of 8 column tiles per row tile on 148 CTAs: round robin vs LPT
        const int nt_ = (int)f->u_off.size() - 1, items = nt_ * 8, G = 148;
        std::vector<double> rr(G, 0.0), lpt(G, 0.0);
        std::vector<std::pair<int, int>> it;
        for (int i = 0; i < items; ++i) {
          const int c = f->u_off[i / 8 + 1] - f->u_off[i / 8] + 2;  // + ~2 blocks of per-item drain / epilogue
          rr[i % G] += c;
          it.push_back({c, i});
        }
        std::sort(it.begin(), it.end(), [](auto& a, auto& b) { return a.first > b.first; });
        for (auto& p : it) *std::min_element(lpt.begin(), lpt.end()) += p.first;
        double tot = 0;
        for (double v : rr) tot += v;
        std::fprintf(stderr, "[lfm]   148 CTAs: mean %.1f, round-robin max %.1f, LPT max %.1f (block units)\n", tot / G,
                     *std::max_element(rr.begin(), rr.end()), *std::max_element(lpt.begin(), lpt.end()));
      }
    }
    for (int G : {4, 8, 16})
      std::fprintf(stderr, "[lfm] MSEG density with %2d-row groups: ca1n %.3f  cf1n %.3f  ca0 %.3f  cf0 %.3f\n", G,
                   mseg_density(cp.ca1n, G), mseg_density(cp.cf1n, G), mseg_density(cp.ca[0], G), mseg_density(cp.cf[0], G));
  }
  // collapsed path
  sep_init(cp.fwd_c, &cp.cf[0], &cp.cf[1], nx, ny, 1, (float)(c1 * c3));
  for (int n = 0; n < nz; ++n) sep_add(cp.fwd_c, n * nslice, n, n, 1.f);
  sep_close_output(cp.fwd_c);
  // collapsed adjoint in two passes (the transposed composite spans ~10 lenslet sub-images, too wide to
  // stage in 2D): Z_n = C_t,n^T y along t (s untouched), then x_n = C_s,n^T Z_n along s.
  make_identity(cp.id_s, ndet[0]);
  make_identity(cp.id_vt, ny);
  // The intermediate Z of both two-pass orders is slice-interleaved: row (vt, n) at (vt*nz + n)*ndet_s.
  // adjoint pass t: one term over the rows-by-slice family (4 neighbouring slices of one voxel row per
  // G4 group: nearly identical bands, so the MSEG segments are ~95% dense)
  sep_init(cp.adj_c1, &cp.id_s, &cp.ca1n, ndet[0], ndet[1], 1, 1.f);
  cp.adj_c1.s_ident = 1;
  sep_add(cp.adj_c1, 0, 0, 0, 1.f);
  sep_close_output(cp.adj_c1);
  // adjoint pass s: x_n = C_s,n^T Z_n, reading slice n's rows at pitch nz*ndet_s
  sep_init(cp.adj_c2, &cp.ca[0], &cp.id_vt, ndet[0], ny, nz, (float)(c1 * c3));
  cp.adj_c2.src_pitch = (long long)nz * ndet[0];
  for (int n = 0; n < nz; ++n) {
    sep_add(cp.adj_c2, (long long)n * ndet[0], n, 0, 1.f);
    sep_close_output(cp.adj_c2);
  }
  // collapsed forward in two passes: U_n = X_n C_{s,n}^T (all slices, t identity, written interleaved),
  // then y = C_t U over the cols-by-slice family: the slice sum is one long band per detector row
  sep_init(cp.fwd_c1, &cp.cf[0], &cp.id_vt, nx, ny, nz, 1.f);
  cp.fwd_c1.out_pitch = (long long)nz * ndet[0];
  cp.fwd_c1.out_stride = ndet[0];
  for (int n = 0; n < nz; ++n) {
    sep_add(cp.fwd_c1, n * nslice, n, 0, 1.f);
    sep_close_output(cp.fwd_c1);
  }
  sep_init(cp.fwd_c2, &cp.id_s, &cp.cf1n, ndet[0], ny * nz, 1, (float)(c1 * c3));
  cp.fwd_c2.s_ident = 1;
  sep_add(cp.fwd_c2, 0, 0, 0, 1.f);
  sep_close_output(cp.fwd_c2);
  // terms >= 1 of a non-separable lenslet stage: their own interleaved t families and t-pass ops (the s passes run
  // on their band_v tables, built at upload); the collapsed path then sums the terms (tcgen05 kernels only)
  for (Component& cm : cp.comps) {
    make_rows_by_slice(cm.ca1n, cm.ca[1]);
    if (nz % 64 == 0 && !std::getenv("LFM_UMMA_ROWS128")) {
      cm.ca1n.u_mode = 1;
      cm.ca1n.u_nz = nz;
    }
    build_umma(cm.ca1n);
    make_cols_by_slice(cm.cf1n, cm.cf[1]);
    build_umma(cm.cf1n);
    sep_init(cm.adj_c1, &cp.id_s, &cm.ca1n, ndet[0], ndet[1], 1, 1.f);
    cm.adj_c1.s_ident = 1;
    sep_add(cm.adj_c1, 0, 0, 0, 1.f);
    sep_close_output(cm.adj_c1);
    sep_init(cm.fwd_c2, &cp.id_s, &cm.cf1n, ndet[0], ny * nz, 1, (float)(c1 * c3));
    cm.fwd_c2.s_ident = 1;
    sep_add(cm.fwd_c2, 0, 0, 0, 1.f);
    sep_close_output(cm.fwd_c2);
  }
  // transposed variants of the s passes (t passes over transposed slices, written back transposed):
  //  fwd_p1: U[(vt,n)][i_s] = sum_vx C_s,n[i_s][vx] xT_n[vx][vt]     (xT_n = x_n transposed, [vx][vt])
  //  adj_a2: x_n[vt][vx]   = sum_j C_s,n^T[vx][j] ZT_n[j][vt]        (ZT_n = Z_n transposed, [j][vt])
  if (ny % 4 == 0) {  // band_m reads whole 16-byte column quads of the transposed slices
  sep_init(cp.fwd_p1, &cp.id_vt, &cp.cf[0], ny, nx, nz, 1.f);
  cp.fwd_p1.s_ident = 1;
  cp.fwd_p1.tout = 1;
  cp.fwd_p1.out_pitch = (long long)nz * ndet[0];
  cp.fwd_p1.out_stride = ndet[0];
  for (int n = 0; n < nz; ++n) {
    sep_add(cp.fwd_p1, n * nslice, 0, n, 1.f);
    sep_close_output(cp.fwd_p1);
  }
  sep_init(cp.adj_a2, &cp.id_vt, &cp.ca[0], ny, ndet[0], nz, (float)(c1 * c3));
  cp.adj_a2.s_ident = 1;
  cp.adj_a2.tout = 1;
  cp.adj_a2.out_pitch = nx;
  cp.adj_a2.out_stride = nslice;
  for (int n = 0; n < nz; ++n) {
    sep_add(cp.adj_a2, (long long)n * ndet[0] * ny, 0, n, 1.f);
    sep_close_output(cp.adj_a2);
  }
  }
  // lf_transport ops: output b = n*K + k (S1 families), b = k (S3 families); scale 1/V^p
  {
    long long dplane = plen ? nfield : npix;
    sep_init(cp.xp_s1f, &cp.s1f[0], &cp.s1f[1], nx, ny, nz * Kv, (float)(1.0 / Vdst));
    for (int n = 0; n < nz; ++n)
      for (int kt = 0; kt < K[1]; ++kt)
        for (int ks = 0; ks < K[0]; ++ks) {
          sep_add(cp.xp_s1f, (long long)(kt * K[0] + ks) * nslice, tab(ks, n), tab(kt, n), 1.f);
          sep_close_output(cp.xp_s1f);
        }
    sep_init(cp.xp_s1a, &cp.s1a[0], &cp.s1a[1], dst[0].n, dst[1].n, nz * Kv, 1.f);
    for (int n = 0; n < nz; ++n) {
      // V^{q_n} per axis = Delta^r * D0 / z_n
      double Vq = (vox_r[0] * d0[0] / std::fabs(zs[n])) * (vox_r[1] * d0[1] / std::fabs(zs[n]));
      for (int kt = 0; kt < K[1]; ++kt)
        for (int ks = 0; ks < K[0]; ++ks) {
          sep_add(cp.xp_s1a, (long long)(kt * K[0] + ks) * dplane, tab(ks, n), tab(kt, n), (float)(1.0 / Vq));
          sep_close_output(cp.xp_s1a);
        }
    }
    if (plen) {
      sep_init(cp.xp_s3f, &cp.s3f[0], &cp.s3f[1], dst[0].n, dst[1].n, Kv, (float)(1.0 / Vmu));
      sep_init(cp.xp_s3a, &cp.s3a[0], &cp.s3a[1], ndet[0], ndet[1], Kv, (float)(1.0 / Vdst));
      for (int kt = 0; kt < K[1]; ++kt)
        for (int ks = 0; ks < K[0]; ++ks) {
          for (int tau = 0; tau < T; ++tau)
            sep_add(cp.xp_s3f, (long long)(kt * K[0] + ks) * nfield, ks * T + tau, kt * T + tau, 1.f);
          sep_close_output(cp.xp_s3f);
          for (int tau = 0; tau < T; ++tau)
            sep_add(cp.xp_s3a, (long long)(kt * K[0] + ks) * npix, ks * T + tau, kt * T + tau, 1.f);
          sep_close_output(cp.xp_s3a);
        }
    }
  }
  SepOp* ops[] = {&cp.fwd_s1, &cp.fwd_s3, &cp.adj_s3, &cp.adj_s1, &cp.fwd_c, &cp.adj_c1, &cp.adj_c2,
                  &cp.xp_s1f, &cp.xp_s1a, &cp.xp_s3f, &cp.xp_s3a, &cp.fwd_c1, &cp.fwd_c2, &cp.fwd_p1, &cp.adj_a2};
  const char* names[] = {"fwd_s1", "fwd_s3", "adj_s3", "adj_s1", "fwd_c", "adj_c1", "adj_c2",
                         "xp_s1f", "xp_s1a", "xp_s3f", "xp_s3a", "fwd_c1", "fwd_c2", "fwd_p1", "adj_a2"};
  const bool dbg = std::getenv("LFM_DEBUG") != nullptr;
  if (dbg) {
    const BandFamily* fams[] = {&cp.s1f[0], &cp.s1f[1], &cp.s1a[0], &cp.s1a[1], &cp.s3f[0], &cp.s3f[1],
                                &cp.s3a[0], &cp.s3a[1], &cp.cf[0],  &cp.cf[1],  &cp.ca[0],  &cp.ca[1]};
    const char* fn[] = {"s1f0", "s1f1", "s1a0", "s1a1", "s3f0", "s3f1", "s3a0", "s3a1", "cf0", "cf1", "ca0", "ca1"};
    for (int i = 0; i < 12; ++i)
      if (fams[i]->st_cols_g4 > 0)
        std::fprintf(stderr, "[lfm] family %-4s G4 density %.3f  (any-nonzero columns only: %.3f)\n", fn[i],
                     fams[i]->st_nnz / (4 * fams[i]->st_cols_g4), fams[i]->st_nnz / (4 * fams[i]->st_cols_nz));
  }
  for (int q = 0; q < 15; ++q) {
    if (!ops[q]->fs) continue;
    if (ops[q]->s_ident && ops[q]->ft->want_mseg && ops[q]->n_is % 4 == 0) {
      // identity s over an MSEG t family: the L2-gather kernel needs no shared memory (autotuned later)
      SepOp& op = *ops[q];
      op.kind = 3; op.ts = 128; op.tt = 16; op.nt = 128; op.nb = 1; op.stage = 0; op.stages = 4;
      fill_sep_geometry(op);
    } else if (!sep_choose_tile(*ops[q])) {
      err = std::string("source footprint of op ") + names[q] + " exceeds shared memory";
      return LFM_E_NOMEM;
    }
    // tuning hook: LFM_FORCE_<op>=ts,tt,nt,nb,stage overrides the cost model (sweeps, tools/)
    std::string env = std::string("LFM_FORCE_") + names[q];
    if (const char* f = std::getenv(env.c_str())) {
      // optional 6th/7th fields: kind (3 = band_m L2 gather over MSEG segments, 5 = band_f flat entries, 8 = band_u
      // tcgen05; identity-s ops only), stages (unroll, or band_u's drain group), MSEG group rows
      int ts, tt, nt, nb, stg, kind = 0, stages = 2, mg = 4, chk = 32;
      if (std::sscanf(f, "%d,%d,%d,%d,%d,%d,%d,%d,%d", &ts, &tt, &nt, &nb, &stg, &kind, &stages, &mg, &chk) >= 5) {
        SepOp& op = *ops[q];
        op.ts = ts; op.tt = tt; op.nt = nt; op.nb = nb; op.stage = stg; op.kind = kind; op.stages = stages; op.mgrp = mg;
        fill_sep_geometry(op);
        if (kind >= 1) {
          bool ok = (kind == 3 || kind == 5 || kind == 8) && op.s_ident && op.n_is % 4 == 0 && op.ft->want_mseg &&
                    (mg == 4 || (kind == 3 && mg == 8 && !op.ft->m8_off.empty())) &&
                    (kind != 5 || !op.ft->f_off.empty()) &&
                    (kind != 8 || (!op.ft->u_off.empty() && !op.tout && op.n_out == 1 && op.terms.size() == 1));
          for (const Term& t : op.terms) ok &= (t.src_off % 4) == 0;
          if (!ok) { err = env + ": kernel kind not applicable"; return LFM_E_INVALID; }
        } else if (sep_smem(op, nb) > (size_t)220 * 1024) {
          err = env + ": shared memory too large";
          return LFM_E_INVALID;
        }
      }
    }
    if (dbg)
      std::fprintf(stderr, "[lfm] %-7s nt %3d tile %3dx%-3d nb %d stage %d fs %4d ft %4d wt %5d gmax_s %3d gmax_t %3d smem %6zu fma %.3g\n",
                   names[q], ops[q]->nt, ops[q]->ts, ops[q]->tt, ops[q]->nb, ops[q]->stage, ops[q]->fs_max, ops[q]->ft_max,
                   ops[q]->wt_max, ops[q]->fs->gmax, ops[q]->ft->gmax, sep_smem(*ops[q], ops[q]->nb), ops[q]->fma_alg);
  }

  // algorithmic work and bytes per A_forward
  double rot_bytes = 0;
  for (int p = 0; p < 3; ++p)
    if (cp.rot[p].active) rot_bytes += 8.0 * info.n_vox;
  info.fma_alg[0] = cp.fwd_s1.fma_alg + (plen ? cp.fwd_s3.fma_alg : 0.0);
  info.fma_alg[1] = cp.fwd_c.fma_alg;
  {
    double nnz_f = 0, nnz_a = 0;
    for (size_t i = 0; i < cp.cf1n.cnt.size(); ++i) nnz_f += cp.cf1n.cnt[i];
    for (size_t i = 0; i < cp.ca1n.cnt.size(); ++i) nnz_a += cp.ca1n.cnt[i];
    info.fma_stage[0] = nnz_f * ndet[0];
    info.fma_stage[1] = nnz_a * ndet[0];
    info.mma_stage[0] = 3.0 * 128 * 16 * (double)cp.cf1n.u_k0.size() * ndet[0];
    info.mma_stage[1] = 3.0 * 128 * 16 * (double)cp.ca1n.u_k0.size() * ndet[0];
    double nnz_sf = 0, nnz_sa = 0;
    for (int v : cp.cf[0].cnt) nnz_sf += v;
    for (int v : cp.ca[0].cnt) nnz_sa += v;
    info.fma_spass[0] = nnz_sf * ny;
    info.fma_spass[1] = nnz_sa * ny;
  }
  info.bytes_alg[0] = 4.0 * info.n_vox + rot_bytes + (plen ? 8.0 * Kv * nfield : 0.0) + 4.0 * npix;
  info.bytes_alg[1] = 4.0 * info.n_vox + rot_bytes + 4.0 * npix;

  // workspace: two rotation buffers, the per-view fields, residual/scratch, reduction partials
  cp.ws_rot = (size_t)info.n_vox * 4;
  cp.ws_fields = (size_t)(Kv * (plen ? nfield : 0)) * 4;
  cp.ws_z = (size_t)nz * ny * ndet[0] * 4;
  size_t scratch = std::max((size_t)npix * 4, (size_t)info.n_vox * 4);
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  info.ws_bytes = 2 * al(cp.ws_rot) + al(cp.ws_fields) + al(scratch) + al(4096 * 8 * 4);
  return LFM_OK;
}

}  // namespace lfm
