/* liblfm -- B200-native (sm_100a) matrix-free light-transport system model for plenoptic
 * chemiluminescence tomography (arXiv 1812.03358).  C ABI.
 *
 * Citation keys: "P:n" = line n of the paper text; equation labels are the
 * paper's own.  Readings of silent/garbled passages (Z1..Z24) are listed in DESIGN.md.
 *
 * Conventions for every call:
 *  - Units are millimetres; slopes are dimensionless.
 *  - Every data buffer is fp32, caller-allocated and caller-owned, on the plan's CUDA
 *    device.  The plan owns only its coefficient tables.  Workspace `ws` (>= ws_bytes from
 *    lfm_plan_info, 256-byte aligned) is caller-owned scratch; a call may overwrite all of it.
 *  - Apply calls are asynchronous and ordered on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream); none synchronises the host.  A plan is immutable after
 *    creation, so concurrent applies on different streams with distinct workspaces are safe.
 *  - Layouts: a volume is x fastest, then y, then z (nx*ny*nz floats, eqn,voxel P:1036-1044);
 *    a light-field plane is s fastest then t; multi-view fields are view-major with
 *    view index k = k_t*K_s + k_s; a detector image is n_t rows of n_s pixels.
 *  - Data buffers must be 16-byte aligned (the tensor-core t passes move rows by TMA);
 *    cudaMalloc and PyTorch allocations are.  A misaligned buffer gives LFM_E_INVALID.
 *  - Outputs are overwritten unless an `accumulate` argument is non-zero.
 *  - Errors: every call returns an lfm_status and never throws; lfm_last_error() gives a
 *    thread-local message naming the failing camera, axis or block.
 *    Invalid arguments are detected before any device work is enqueued.
 */
#ifndef LFM_H
#define LFM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LFM_OK = 0,
  LFM_E_INVALID = 1,    /* null pointer, bad index/plane id, bad dims, fill > 1, ws too small */
  LFM_E_SINGULAR = 2,   /* |det| <= 1e-12 of an optical block, zero focal length */
  LFM_E_DEGENERATE = 3, /* b_q = 0 or lambda = 0 (plane on/conjugate to the angular plane),
                           rotation outside the shear-decomposable set (>= 45 deg) */
  LFM_E_MISMATCH = 4,   /* unsupported plane pair for lf_transport */
  LFM_E_ZERO_DATA = 5,  /* ||W^1/2 y_c|| = 0 for a camera c >= 2 (gain undefined) */
  LFM_E_NONFINITE = 6,  /* non-finite cost */
  LFM_E_CUDA = 7,       /* a CUDA runtime error (message has the CUDA string) */
  LFM_E_NOMEM = 8       /* device allocation of plan tables failed */
} lfm_status;

typedef enum { LFM_FWD = 0, LFM_ADJ = 1 } lfm_dir;
typedef enum { LFM_PILLBOX = 0, LFM_DIRAC = 1 } lfm_basis;            /* angular basis a */
typedef enum { LFM_SINGLE = 0, LFM_PLENOPTIC = 1 } lfm_camera_type;   /* §2.6 */
/* Evaluation order of A_c (both exact re-associations of the same operator):
 *  LFM_PATH_PER_VIEW  : the paper's factored chain (eqn,plenoptic,factor P:1077-1097): per view k,
 *                       slices -> lenslet array (S1), then mask + lenslets -> detector (S3).
 *  LFM_PATH_COLLAPSED : the sum over the tensor angular grid folded into one separable operator per
 *                       slice, C_n = sum_k S_k B_{k,n} per axis; same A, fewer FMAs. */
typedef enum { LFM_PATH_PER_VIEW = 0, LFM_PATH_COLLAPSED = 1 } lfm_path;

typedef struct { int nx, ny, nz; double dx, dy, dz; } lfm_volume; /* voxel grid centred on 0 */

typedef struct {
  int type;                 /* lfm_camera_type */
  int basis;                /* lfm_basis */
  double f_main;            /* main-lens focal length */
  double ap_s, ap_t;        /* square aperture sides on the angular plane (= main lens) */
  double d_scene;           /* main lens -> volume centre (D_scene) */
  int k_s, k_t;             /* angular samples per axis, K = k_s*k_t, tensor grid (Z4) */
  double d_det;             /* single-lens: lens -> detector distance D */
  double d_mu_m;            /* plenoptic: main lens -> lenslet array (D_mu_m) */
  double d_d_mu;            /* plenoptic: lenslet array -> detector (D_d_mu) */
  double f_mu;              /* plenoptic: lenslet focal length */
  double fill;              /* plenoptic: lenslet square aperture side / pitch, 0 < fill <= 1 */
  int nl_s, nl_t;           /* plenoptic: lenslet grid; pitch = n_s*px_s/nl_s */
  int n_a;                  /* plenoptic: array-plane cells per lenslet per axis (Z11) */
  int n_s, n_t;             /* detector pixels */
  double px_s, px_t;        /* detector pitch */
  double R[9];              /* pose Theta, row-major, p = Theta p_r, residual < 45 deg */
  int lens_layout;          /* plenoptic: 0 rectangular lenslet grid; 1 hexagonal: odd lenslet rows (along t)
                               shifted by pitch_s/2 along s and holding nl_s - 1 lenslets (reading R12) */
  int aperture;             /* plenoptic: 0 square lenslet apertures (side fill*pitch per axis); 1 circular: array
                               cells whose centres lie strictly inside the disk of diameter fill*pitch_s (the
                               occluder rasterised onto the array grid, eqn,occlusion P:915-927; reading R13).
                               Overlapping apertures give LFM_E_INVALID. */
} lfm_camera;

typedef struct {
  lfm_volume vol;
  int n_cam;
  const lfm_camera* cam;    /* n_cam entries, copied by lfm_plan_create */
  int n_subsets;            /* view subsets for the ordered-subsets gradient (sec,subset P:360-388):
                               0 or 1 = none; M > 1 builds, per camera, subset m = every M-th view of the
                               lexicographically ordered angular plane starting at m (k = k_t*K_s + k_s) */
} lfm_geometry;

typedef struct lfm_plan_s* lfm_plan;

/* Per-camera plan facts (lfm_plan_info). */
typedef struct {
  int type, basis;
  int nx, ny, nz;           /* volume dims (rotated grid has the same dims) */
  long long n_vox;
  int n_s, n_t;             /* detector */
  long long n_pix;
  int k_s, k_t, n_views;
  int n_as, n_at;           /* lenslet-array plane cells (0 for single-lens) */
  int plane_array;          /* lf_transport plane id of the array plane (-1 if none) = nz */
  int plane_detector;       /* plane id of the detector = nz + 1 */
  double vox_r[3];          /* rotated voxel sizes Delta/D */
  double rot_D[3];          /* D_Theta */
  double shear[6];          /* a_zx a_zy a_xy a_xz a_yx a_yz (eqn,rot,decomp) */
  int rot_passes;           /* bitmask of non-identity rotation stages: 1=z 2=x 4=y shear passes, 8=quarter-turn
                               relabelling applied first (poses beyond 45 deg, reading R7) */
  int rot_perm[9];          /* that relabelling P (signed permutation, row-major; identity if bit 8 is clear):
                               Theta = P D S_z S_x S_y */
  int taps_s1, taps_s3, taps_c;  /* padded band widths of the S1, S3 and collapsed tables */
  size_t ws_bytes;          /* workspace needed by every apply call on this camera */
  size_t table_bytes;       /* device bytes of this camera's tables */
  double fma_alg[2];        /* algorithmic FMAs (plan nnz) per A_forward per path [per_view, collapsed] */
  double bytes_alg[2];      /* algorithmic HBM bytes per A_forward per path */
  double fma_stage[2];      /* algorithmic FMAs (non-zeros x columns) of one launch of stage
                               LFM_STAGE_FWD_T / LFM_STAGE_ADJ_T (lfm_A_stage) */
  double mma_stage[2];      /* tensor-core MACs one launch of those stages issues when it runs on the tcgen05
                               kernel (3 products x dense 128 x 16 blocks x columns) */
  int kind_stage[2];        /* kernel the autotuner chose for those stages (8 = tcgen05 band_u, 5 = band_f, ...) */
  double fma_spass[2];      /* algorithmic FMAs of one launch of LFM_STAGE_FWD_S / LFM_STAGE_ADJ_S (the collapsed
                               path's s passes: non-zeros of C_s,n summed over slices x ny voxel rows) */
  int subset_collapsed;     /* how many of the plan's view subsets run on the collapsed path (tensor-product
                               subsets, lfm_A_forward_subset); the others use the per-view path */
  int s3_terms;             /* separable terms T of the lenslet stage (1 for a rectangular grid with square
                               apertures; hexagonal layouts / circular apertures: S_k = sum_tau S^tau_ks (x) S^tau_kt,
                               reading R12).  S3 table ids index k*T + tau; the collapsed path sums T terms. */
  int f16_stage[2];         /* 1 when the collapsed path's forward / adjoint t pass runs in the 2xFP16 form
                               (fp16 hi + lo operands, kind::f16 MMAs), 0 for 3xTF32 */
} lfm_info;

/* Table ids for lfm_plan_export_table (bit-exact comparison with the oracle in tests).
 * For an id with `index` = (k_axis * nz + n) (S1 families) or k_axis (S3 families) or n (collapsed)
 * or pass (shear), the export writes either int32 [rows] (START/LEN) or fp64 [rows*taps] (W64). */
typedef enum {
  LFM_TAB_S1F_START = 0, LFM_TAB_S1F_LEN = 1, LFM_TAB_S1F_W64 = 2,   /* slice n -> array/detector  */
  LFM_TAB_S1A_START = 3, LFM_TAB_S1A_LEN = 4, LFM_TAB_S1A_W64 = 5,   /* array/detector -> slice n  */
  LFM_TAB_S3F_START = 6, LFM_TAB_S3F_LEN = 7, LFM_TAB_S3F_W64 = 8,   /* array -> detector (masked) */
  LFM_TAB_S3A_START = 9, LFM_TAB_S3A_LEN = 10, LFM_TAB_S3A_W64 = 11, /* detector -> array (masked) */
  LFM_TAB_CF_START = 12, LFM_TAB_CF_LEN = 13, LFM_TAB_CF_W64 = 14,   /* collapsed slice n -> detector */
  LFM_TAB_ROT_MLO = 15, LFM_TAB_ROT_W64 = 16,                        /* shear pass lines (fwd) */
  LFM_TAB_SCALARS = 17                                               /* fp64 [8]: see lfm_plan.cpp */
} lfm_table_id;

/* --- plan --------------------------------------------------------------------------------- */
/* Build every camera's optics chain (§2.1), rotation factors (closed form of eqn,rot,decomp),
 * 1D band tables of the L2 transport entries (eqn,xport,int; closed form of the missing
 * tab,pillbox/tab,dirac) in fp64, rounded once to fp32, and upload them to
 * `cuda_device`.  Host work, not on the hot path.  *out receives the plan (NULL on error).
 * cuda_device = -1 builds a host-only plan (no CUDA calls; only lfm_plan_info and
 * lfm_plan_export_table are valid on it -- used by the CPU test suite). */
lfm_status lfm_plan_create(const lfm_geometry* g, int cuda_device, lfm_plan* out);
lfm_status lfm_plan_destroy(lfm_plan p);
lfm_status lfm_plan_info(lfm_plan p, int cam, lfm_info* out);
/* axis 0 = s, 1 = t.  `bytes` must equal the table size exactly (query with host_dst = NULL,
 * which stores the needed size in *bytes_needed). */
lfm_status lfm_plan_export_table(lfm_plan p, int cam, int table_id, int axis, int index,
                                 void* host_dst, size_t bytes, size_t* bytes_needed);

/* --- the hot path ------------------------------------------------------------------------- */
/* Light transport between two planes of camera `cam`, all K views (eqn,xport,sep):
 *   dst_k = (1/V^p) B^{pq}_k src_k,   B = B_s (x) B_t as a t-pass then an s-pass.
 * Plane ids: 0..nz-1 = slices of the rotated volume, nz = lenslet array (plenoptic),
 * nz+1 = detector.  Supported pairs: slice<->array and array<->detector (plenoptic; the
 * detector field is the masked superposition over lenslets), slice<->detector
 * (single-lens).  (q,p) gives the V-scaled adjoint: (V^q/V^p) lf_transport(q,p) is the
 * adjoint of lf_transport(p,q).  src: [K][n_t(q)][n_s(q)], dst: [K][n_t(p)][n_s(p)]. */
lfm_status lfm_lf_transport(lfm_plan p, int cam, int dst_plane, int src_plane, const float* src,
                            float* dst, void* ws, size_t ws_bytes, void* stream);

/* Resample the volume into camera cam's rotated frame: x^r = E^y E^x E^z x (LFM_FWD) or its
 * adjoint E^zT E^xT E^yT (LFM_ADJ) (eqn,rot,toeplitz).  in/out: nx*ny*nz floats,
 * must not alias. */
lfm_status lfm_vol_rotate(lfm_plan p, int cam, int dir, const float* in, float* out,
                          int accumulate, void* ws, size_t ws_bytes, void* stream);

/* dst += src over n floats (the sum over cameras of the backprojections, sum_c A_c^T r_c in the PWLS gradient
 * eqn,pls P:299-317, when the cameras run concurrently on their own streams into private volumes).  dst and
 * src must not alias; n >= 0. */
lfm_status lfm_vol_accumulate(const float* src, float* dst, long long n, void* stream);

/* y = A_c x (rotation, slice collapse, camera; §3.2).  x: n_vox, y: n_pix. */
lfm_status lfm_A_forward(lfm_plan p, int cam, int path, const float* x, float* y,
                         void* ws, size_t ws_bytes, void* stream);
/* x (+)= A_c^T y, each transport evaluated as the scaled forward transport in the opposite
 * direction (B^{pq} = (B^{qp})^T). */
lfm_status lfm_A_adjoint(lfm_plan p, int cam, int path, const float* y, float* x, int accumulate,
                         void* ws, size_t ws_bytes, void* stream);

/* Detector-row sharding: rows [row0, row1) of y = A_c x (other rows of y may also
 * be written with their correct values where an output tile straddles the range), and
 * x (+)= A_c^T P y where P keeps only rows [row0, row1) of y (treated as zero elsewhere).  Summing
 * lfm_A_adjoint_rows over a partition of the rows gives lfm_A_adjoint.  0 <= row0 < row1 <= n_t. */
lfm_status lfm_A_forward_rows(lfm_plan p, int cam, int path, int row0, int row1, const float* x, float* y,
                              void* ws, size_t ws_bytes, void* stream);
lfm_status lfm_A_adjoint_rows(lfm_plan p, int cam, int path, int row0, int row1, const float* y, float* x,
                              int accumulate, void* ws, size_t ws_bytes, void* stream);
/* Detector windows (rows [row0, row1) x columns [col0, col1)), the shards of the multi-GPU partition:
 * lfm_A_forward_window writes y on the window (other entries of partially covered tiles may also be written, with
 * their correct values); lfm_A_adjoint_window gives x (+)= A_c^T P y with P keeping only the window of y.  Summing
 * the adjoint over a partition of the detector into windows gives lfm_A_adjoint.  On the collapsed tcgen05 path a
 * column window restricts every kernel to the window's 256-column tiles (the s passes act column by column, the t
 * passes tile by tile; the forward t pass splits K when the window leaves most SMs idle, with partial sums in the
 * workspace added in a fixed order); elsewhere the column window is applied by masking y.
 * 0 <= row0 < row1 <= n_t, 0 <= col0 < col1 <= n_s, else LFM_E_INVALID. */
lfm_status lfm_A_forward_window(lfm_plan p, int cam, int path, int row0, int row1, int col0, int col1, const float* x,
                                float* y, void* ws, size_t ws_bytes, void* stream);
lfm_status lfm_A_adjoint_window(lfm_plan p, int cam, int path, int row0, int row1, int col0, int col1, const float* y,
                                float* x, int accumulate, void* ws, size_t ws_bytes, void* stream);

/* View-subset operators (sec,subset, eqn,subset P:366-379, reading Z19): with S_m the plan's subset m,
 *   y = (K/|S_m|) sum_{k in S_m} A_ck x           (lfm_A_forward_subset)
 *   x (+)= (K/|S_m|) sum_{k in S_m} A_ck^T y      (lfm_A_adjoint_subset)
 * evaluated on the collapsed path when S_m is a tensor product S_s x {all k_t} (M divides K_s: the s composite is
 * re-collapsed over S_s, the t pass is the full one; lfm_info.subset_collapsed counts these), else on the per-view
 * path.  0 <= subset < n_subsets of the
 * plan (LFM_E_INVALID otherwise, also when the plan has no subsets).  Same buffers and workspace as
 * lfm_A_forward / lfm_A_adjoint. */
lfm_status lfm_A_forward_subset(lfm_plan p, int cam, int subset, const float* x, float* y, void* ws, size_t ws_bytes,
                                void* stream);
lfm_status lfm_A_adjoint_subset(lfm_plan p, int cam, int subset, const float* y, float* x, int accumulate, void* ws,
                                size_t ws_bytes, void* stream);

/* Single stages of the collapsed two-pass path (NEXT-1), for measuring
 * the dominant kernels in isolation.  Each stage is ONE kernel launch and reads / writes the
 * slice-interleaved intermediate Z that the workspace holds after a full call:
 *   LFM_STAGE_FWD_T: y = sum over (vt, n) of C_t[i_t][(vt, n)] Z[(vt, n)][:]  (Z from the last
 *                    lfm_A_forward of this camera with this workspace; `in` unused, `out` = y);
 *   LFM_STAGE_ADJ_T: Z[(vt, n)][:] = sum over i_t of C_t,n^T[vt][i_t] y[i_t][:]  (`in` = y; `out` unused,
 *                    Z is left in the workspace).
 * Status LFM_E_INVALID if the camera's collapsed path is not in its two-pass form. */
/*   LFM_STAGE_FWD_S: Z[(vt, n)][:] = sum_vx x^r_n[vt][vx] C_s,n[:][vx]  (`in` = x^r, the rotated volume;
 *                    `out` unused, Z is left in the workspace for LFM_STAGE_FWD_T);
 *   LFM_STAGE_ADJ_S: out_n[vt][vx] = c sum_i C_s,n^T[vx][i] Z[(vt, n)][i]  (Z from the last lfm_A_adjoint or
 *                    LFM_STAGE_ADJ_T with this workspace; `out` = the rotated-frame volume, overwritten). */
enum { LFM_STAGE_FWD_T = 0, LFM_STAGE_ADJ_T = 1, LFM_STAGE_FWD_S = 2, LFM_STAGE_ADJ_S = 3 };
lfm_status lfm_A_stage(lfm_plan p, int cam, int stage, const float* in, float* out, void* ws, size_t ws_bytes,
                       void* stream);

/* --- PWLS with the camera gains minimised out (eqn,pls P:299-317; App. A) --------
 * Weights are absorbed (A~ = W^1/2 A, y~ = W^1/2 y); w = diag(W_c) >= 0.
 * Phase 1, per camera: stats3_dev[0..2] = [y'W(Ax), y'Wy, (Ax)'W(Ax)] in fp64 (deterministic
 * two-level reduction).  Between phases a multi-GPU caller all-reduces the stats. */
lfm_status lfm_pwls_stats(lfm_plan p, int cam, const float* Ax, const float* y, const float* w,
                          double* stats3_dev, void* ws, size_t ws_bytes, void* stream);
/* gamma_dev[c] = 1 for c = 0, else stats[c][0]/stats[c][1] (eqn,optimal,gain P:110-114).
 * stats_dev: n_cam*3 doubles.  Returns LFM_E_ZERO_DATA via *flag_dev != 0 (checked by the caller,
 * no host sync here). */
lfm_status lfm_pwls_gains(lfm_plan p, const double* stats_dev, double* gamma_dev, int* flag_dev,
                          void* stream);
/* Phase 2: grad = sum_c A_c^T W_c (A_c x - gamma_c y_c) + beta * sum_{l in N_j}(x_j - x_l) + nu
 * over the cameras [cam0, cam1) of this rank (a multi-GPU caller all-reduces grad afterwards and
 * adds the regulariser on one rank only: include_reg).  cost_dev (nullable): fp64 [2] =
 * [sum_c 1/2||.||^2_W, nu*sum x + R(x)].  Ax[c], y[c], w[c] are device pointers per camera.
 * subset >= 0: the view-subset gradient of eqn,subset (reading Z19): A_c^T is replaced by
 * (K/|S|) sum_{k in S} A_ck^T and Ax[c] must be the subset prediction of lfm_A_forward_subset; `path`
 * is then ignored.  subset < 0: the exact gradient on `path`.
 * Non-finite cost: when cost_dev is non-NULL (and `stream` is not capturing a graph) the call
 * waits for the stream, reads the cost and returns LFM_E_NONFINITE if either part is NaN or infinite (grad and
 * cost_dev are still written).  Pass cost_dev = NULL for a call that never synchronises.
 * include_reg bit 0: add the regulariser term; bit 1 (LFM_GRAD_ACCUMULATE): grad already holds a partial
 * gradient (other cameras' terms, computed concurrently on other streams): every term of this call is added to
 * it and nothing is zeroed -- so cameras split over streams and summed in camera order, then a call with
 * cam0 == cam1 and include_reg = 3, give the same sums in the same order as one call over all cameras.
 * LFM_GRAD_ACCUMULATE with cost_dev != NULL is LFM_E_INVALID. */
#define LFM_GRAD_ACCUMULATE 2
lfm_status lfm_pwls_grad(lfm_plan p, int path, int subset, int cam0, int cam1, const float* x,
                         const float* const* y, const float* const* w, const float* const* Ax,
                         const double* gamma_dev, float beta, float nu, int include_reg,
                         float* grad, double* cost_dev, void* ws, size_t ws_bytes, void* stream);
/* d = sum_c A_c^T W_c A_c 1 + 36*beta, floored at 1e-12 (App. A; constant 36 per
 * reading Z16).  mode bit LFM_MAJ_SUM: overwrite d with the partial sum over cameras [cam0, cam1);
 * bit LFM_MAJ_FINISH: d = max(d + 36 beta, 1e-12).  One GPU: mode = SUM|FINISH.  Multi-GPU: SUM on
 * every rank, all-reduce d, then FINISH. */
#define LFM_MAJ_SUM 1
#define LFM_MAJ_FINISH 2
lfm_status lfm_majoriser(lfm_plan p, int path, int cam0, int cam1, const float* const* w,
                         float beta, int mode, float* d, void* ws, size_t ws_bytes, void* stream);
/* FISTA step (tab,alg missing; reading Z18), elementwise, in place:
 *   x_new = max(0, z - grad/d);  z = x_new + ((t_old - 1)/t_new) (x_new - x);  x = x_new. */
lfm_status lfm_fista_update(lfm_plan p, float* x, float* z, const float* grad, const float* d,
                            double t_old, double t_new, void* stream);

/* Number of CUDA kernels the last apply call on this thread enqueued (for bench accounting). */
int lfm_last_launch_count(void);
const char* lfm_last_error(void);
const char* lfm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LFM_H */
