"""Single-lens and plenoptic camera models on slice-collapsed volumes (paper §2.6, §3).

Conventions (readings Z1-Z13):

* angular plane = main lens; s <-> x^r, t <-> y^r of the camera-aligned
  (rotated) volume; slice n sits z_n = D_scene + (n - (Nz-1)/2) Dz^r in front of the
  lens (object z increases away from the camera, Z13), X^{0q} = R_f o T_{z_n};
* single-lens detector D behind the lens: X^{0d} = T_{-D};
* plenoptic: array plane X^{0a} = T_{-D_mu_m}; lenslet mu (centre c_mu,
  focal f_mu, detector b = D_d_mu behind the array):
  X^{0mu} = T_{-D_mu_m} o R_{f_mu}(c_mu)^{-1} o T_{-b}  (P:1016 writes X^{0a} o R_mu o T_Ddmu);
* mask M_mu: array cell j is open for lenslet mu iff its centre lies in
  [c_mu - fill*pitch/2, c_mu + fill*pitch/2) (rasterised support; Z9/Z10);
  M = sum_mu M_mu;
* slice collapse: w^n_k = Dz^r x^r_n for every view k;
* normalisation: the literal building blocks f^p = B f^q / V^p and
  y = sqrt(V^d) sum_k f^d_k (reading Z7):
    single-lens:  y = (sqrt(V^d)/V^d) sum_k sum_n B^{d q_n}_k Dz x^r_n
    plenoptic, factored order eqn,plenoptic,factor:
      a_k = (1/V^a) sum_n B^{a q_n}_k Dz x^r_n
      y   = sum_k sum_mu (sqrt(V^mu)/V^mu) B^{mu a}_k M_mu a_k
* memory layout of a plane field: array [t, s] (s fastest); the separable
  product (B_s (x) B_t) f acts as  B_t @ F @ B_s^T.

The plenoptic S3 operator per axis S_k = sum_mu B^{mu a}_k M_mu is formed literally
(one transport per lenslet) -- the oracle does not use the adjoint symmetry; its
adjoint is the literal transpose of every factor.

Non-separable lenslet stages (NEXT-4; "hexagonal microlens configuration"; occluders rasterised onto the
array grid, eqn,occlusion P:915-927; readings R12/R13 of DESIGN.md):
* lens_layout 1 (hexagonal): lenslet row j (along t) has its lenslets shifted by +pitch_s/2 when j is odd, and odd
  rows hold nl_s - 1 lenslets (every lenslet inside the array);
* aperture 1 (circular): array cell (j_s, j_t) is open for lenslet mu iff its centre is strictly inside the disk of
  diameter fill * pitch_s about the lenslet centre; aperture 0 keeps the square rule per axis.
Then M_mu is a 2-D mask and the lenslet stage is evaluated literally lenslet by lenslet,
  y = sum_k sum_mu (sqrt(V^mu)/V^mu) B^{d mu}_{k,t} (M_mu .* a_k) (B^{d mu}_{k,s})^T,
each lenslet's transport still separable (the lens is); no term decomposition in the oracle.
"""
import math

import numpy as np
import scipy.sparse as sp

from .optics import compose, invert, lens, translate
from .transport import Plane, angular_centres, basis_volume, transport_dense, transport_sparse

SINGLE, PLENOPTIC = 0, 1


class CameraModel:
    """Camera c acting on its rotated volume x^r (shape (nz, ny, nx), voxel sizes vox_r)."""

    def __init__(self, cam, dims, vox_r, dense=False):
        self.cam = cam
        self.nonsep = False
        self.nx, self.ny, self.nz = dims
        self.vox_r = vox_r
        self.type = cam["type"]
        self.basis = cam["basis"]
        self.ks, self.kt = cam["k_s"], cam["k_t"]
        self.d0 = (cam["ap_s"] / cam["k_s"], cam["ap_t"] / cam["k_t"])
        self.sk = (angular_centres(self.ks, self.d0[0]), angular_centres(self.kt, self.d0[1]))
        self.dz = vox_r[2]
        self.z = [cam["d_scene"] + (n - (self.nz - 1) * 0.5) * self.dz for n in range(self.nz)]
        build = transport_dense if dense else (lambda *a: transport_sparse(*a))
        self._dense = dense
        n_src = (self.nx, self.ny)
        fm = cam["f_main"]
        self.slice_planes = [[Plane(n_src[ax], vox_r[ax], compose(lens(fm), translate(z))) for z in self.z]
                             for ax in range(2)]
        det_n = (cam["n_s"], cam["n_t"])
        det_d = (cam["px_s"], cam["px_t"])
        if self.type == SINGLE:
            self.det_planes = [Plane(det_n[ax], det_d[ax], translate(-cam["d_det"])) for ax in range(2)]
            dst = self.det_planes
            vd = basis_volume(dst[0], self.d0[0]) * basis_volume(dst[1], self.d0[1])
            self.scale_s1 = self.dz * math.sqrt(vd) / vd
            self.scale_s3 = None
        else:
            nl = (cam["nl_s"], cam["nl_t"])
            na = cam["n_a"]
            self.pitch = tuple(det_n[ax] * det_d[ax] / nl[ax] for ax in range(2))
            self.array_planes = [Plane(nl[ax] * na, self.pitch[ax] / na, translate(-cam["d_mu_m"]))
                                 for ax in range(2)]
            b = cam["d_d_mu"]
            self.lenslet_planes = []
            self.masks = []
            for ax in range(2):
                planes, masks = [], []
                ac = self.array_planes[ax].centres()
                for mu in range(nl[ax]):
                    c_mu = (mu - (nl[ax] - 1) * 0.5) * self.pitch[ax]
                    X0 = compose(translate(-cam["d_mu_m"]), compose(invert(lens(cam["f_mu"], c_mu)), translate(-b)))
                    planes.append(Plane(det_n[ax], det_d[ax], X0))
                    half = 0.5 * cam["fill"] * self.pitch[ax]
                    masks.append(((ac >= c_mu - half) & (ac < c_mu + half)).astype(np.float64))
                self.lenslet_planes.append(planes)
                self.masks.append(masks)
            # non-separable lenslet stage (hexagonal layout and/or circular apertures): one entry per lenslet with
            # its centre, per-axis lenslet planes and a 2-D mask over the array grid [t][s]
            self.layout = int(cam.get("lens_layout", 0))
            self.aperture = int(cam.get("aperture", 0))
            self.nonsep = self.layout != 0 or self.aperture != 0 or bool(cam.get("_force_2d", False))
            if self.nonsep:
                ac_s, ac_t = self.array_planes[0].centres(), self.array_planes[1].centres()
                self.lenslets2d = []
                for j in range(nl[1]):
                    odd = self.layout == 1 and j % 2 == 1
                    c_t = (j - (nl[1] - 1) * 0.5) * self.pitch[1]
                    for i in range(nl[0] - (1 if odd else 0)):
                        c_s = (i - (nl[0] - 1) * 0.5 + (0.5 if odd else 0.0)) * self.pitch[0]
                        if self.aperture == 1:
                            r = 0.5 * cam["fill"] * self.pitch[0]
                            m = ((ac_s[None, :] - c_s) ** 2 + (ac_t[:, None] - c_t) ** 2) < r * r
                        else:
                            hs, ht = 0.5 * cam["fill"] * self.pitch[0], 0.5 * cam["fill"] * self.pitch[1]
                            m = ((ac_s[None, :] >= c_s - hs) & (ac_s[None, :] < c_s + hs) &
                                 (ac_t[:, None] >= c_t - ht) & (ac_t[:, None] < c_t + ht))
                        pls = Plane(det_n[0], det_d[0], compose(translate(-cam["d_mu_m"]),
                                                               compose(invert(lens(cam["f_mu"], c_s)), translate(-b))))
                        plt = Plane(det_n[1], det_d[1], compose(translate(-cam["d_mu_m"]),
                                                               compose(invert(lens(cam["f_mu"], c_t)), translate(-b))))
                        self.lenslets2d.append((c_s, c_t, pls, plt, m.astype(np.float64)))
            dst = self.array_planes
            va = basis_volume(dst[0], self.d0[0]) * basis_volume(dst[1], self.d0[1])
            vmu = basis_volume(self.lenslet_planes[0][0], self.d0[0]) * \
                basis_volume(self.lenslet_planes[1][0], self.d0[1])
            self.scale_s1 = self.dz / va
            self.scale_s3 = math.sqrt(vmu) / vmu
        # S1: slice n -> array (plenoptic) or detector (single), per axis, per k_axis, per n
        self.S1 = [[[build(self.slice_planes[ax][n], dst[ax], self.sk[ax][k], self.d0[ax], self.basis)
                     for n in range(self.nz)] for k in range(len(self.sk[ax]))] for ax in range(2)]
        # non-separable lenslet stage: per view and lenslet the two 1D transports (literal, no symmetry)
        if self.type == PLENOPTIC and self.nonsep:
            self.S3 = None
            self.S3_2d = {}
            for ks in range(len(self.sk[0])):
                for kt in range(len(self.sk[1])):
                    self.S3_2d[ks, kt] = [
                        (build(self.array_planes[0], pls, self.sk[0][ks], self.d0[0], self.basis),
                         build(self.array_planes[1], plt, self.sk[1][kt], self.d0[1], self.basis), m)
                        for (_, _, pls, plt, m) in self.lenslets2d]
        # S3: array -> detector through every lenslet, masked: S_k = sum_mu B^{mu a}_k M_mu
        if self.type == PLENOPTIC and not self.nonsep:
            self.S3 = []
            for ax in range(2):
                per_k = []
                for k in range(len(self.sk[ax])):
                    acc = None
                    for mu, pl in enumerate(self.lenslet_planes[ax]):
                        B = build(self.array_planes[ax], pl, self.sk[ax][k], self.d0[ax], self.basis)
                        term = B @ (np.diag(self.masks[ax][mu]) if dense else sp.diags(self.masks[ax][mu]))
                        acc = term if acc is None else acc + term
                    per_k.append(acc if dense else sp.csr_matrix(acc))
                self.S3.append(per_k)

    @property
    def n_pix(self):
        return self.cam["n_s"] * self.cam["n_t"]

    # ---- matrix-free fp64 forward / adjoint (literal factored order, literal transposes) ----
    def _views(self, views):
        return [(ks, kt) for kt in range(self.kt) for ks in range(self.ks)] if views is None else views

    def forward(self, xr, views=None):
        """y = A x^r; `views` (list of (k_s, k_t)) restricts the sum over k to a sample (bench timing)."""
        xr = np.asarray(xr, np.float64).reshape(self.nz, self.ny, self.nx)
        y = np.zeros((self.cam["n_t"], self.cam["n_s"]))
        for ks, kt in self._views(views):
            acc = np.zeros((self.S1[1][kt][0].shape[0], self.S1[0][ks][0].shape[0]))
            for n in range(self.nz):
                acc += self.S1[1][kt][n] @ (xr[n] @ self.S1[0][ks][n].T)
            acc *= self.scale_s1
            if self.type == PLENOPTIC and self.nonsep:
                for Bs, Bt, m in self.S3_2d[ks, kt]:
                    y += self.scale_s3 * (Bt @ ((m * acc) @ Bs.T))
            elif self.type == PLENOPTIC:
                y += self.scale_s3 * (self.S3[1][kt] @ (acc @ self.S3[0][ks].T))
            else:
                y += acc
        return y

    def adjoint(self, y, views=None):
        y = np.asarray(y, np.float64).reshape(self.cam["n_t"], self.cam["n_s"])
        g = np.zeros((self.nz, self.ny, self.nx))
        for ks, kt in self._views(views):
            if self.type == PLENOPTIC and self.nonsep:
                a = 0.0
                for Bs, Bt, m in self.S3_2d[ks, kt]:
                    a = a + m * (Bt.T @ (y @ Bs))
                a = self.scale_s3 * a
            elif self.type == PLENOPTIC:
                a = self.scale_s3 * (self.S3[1][kt].T @ (y @ self.S3[0][ks]))
            else:
                a = y
            for n in range(self.nz):
                g[n] += self.scale_s1 * (self.S1[1][kt][n].T @ (a @ self.S1[0][ks][n]))
        return g

    # ---- single outputs, one by one (full-size parity on sampled outputs; same factored sums as above) ----
    def forward_at(self, xr, pixels):
        """y[i_t, i_s] = sum_k sum_n (row i of the camera factors) x^r_n for each (i_t, i_s) in `pixels`:
        plenoptic y_i = c3 sum_k (S3t_kt[i_t] c1 S1t_kt,n) x^r_n (S3s_ks[i_s] S1s_ks,n)^T summed over n, the
        factored chain of forward() restricted to one detector pixel."""
        if self.type == PLENOPTIC and self.nonsep:
            raise NotImplementedError("forward_at: separable lenslet stages only")
        xr = np.asarray(xr, np.float64).reshape(self.nz, self.ny, self.nx)
        out = np.zeros(len(pixels))
        for p, (it, i_s) in enumerate(pixels):
            acc = 0.0
            for n in range(self.nz):
                if self.type == PLENOPTIC:
                    rt = np.stack([np.asarray((self.S3[1][kt][it:it + 1] @ self.S1[1][kt][n]).todense()).ravel()
                                   for kt in range(self.kt)])
                    rs = np.stack([np.asarray((self.S3[0][ks][i_s:i_s + 1] @ self.S1[0][ks][n]).todense()).ravel()
                                   for ks in range(self.ks)])
                else:
                    rt = np.stack([self.S1[1][kt][n][it].toarray().ravel() for kt in range(self.kt)])
                    rs = np.stack([self.S1[0][ks][n][i_s].toarray().ravel() for ks in range(self.ks)])
                acc += np.sum(rt @ xr[n] @ rs.T)
            out[p] = acc * self.scale_s1 * (self.scale_s3 if self.type == PLENOPTIC else 1.0)
        return out

    def adjoint_at(self, y, voxels):
        """(A^T y)[n, v_t, v_x] of the rotated frame for each (n, v_t, v_x) in `voxels`: the literal transposes
        of adjoint(), evaluated at single voxels from the per-view array fields a_k = c3 S3t_kt^T y S3s_ks."""
        if self.type == PLENOPTIC and self.nonsep:
            raise NotImplementedError("adjoint_at: separable lenslet stages only")
        y = np.asarray(y, np.float64).reshape(self.cam["n_t"], self.cam["n_s"])
        fields = {}
        for ks in range(self.ks):
            for kt in range(self.kt):
                fields[ks, kt] = self.scale_s3 * (self.S3[1][kt].T @ (y @ self.S3[0][ks])) \
                    if self.type == PLENOPTIC else y
        out = np.zeros(len(voxels))
        for p, (n, vt, vx) in enumerate(voxels):
            acc = 0.0
            for (ks, kt), a in fields.items():
                ct = self.S1[1][kt][n][:, vt].toarray().ravel()
                cs = self.S1[0][ks][n][:, vx].toarray().ravel()
                acc += ct @ a @ cs
            out[p] = self.scale_s1 * acc
        return out

    def array_fields(self, xr):
        """Plenoptic intermediate a_k (K, n_at, n_as) of the factored chain (for S1-stage parity)."""
        xr = np.asarray(xr, np.float64).reshape(self.nz, self.ny, self.nx)
        out = []
        for kt in range(self.kt):
            for ks in range(self.ks):
                acc = 0.0
                for n in range(self.nz):
                    acc = acc + self.S1[1][kt][n] @ (xr[n] @ self.S1[0][ks][n].T)
                out.append(self.scale_s1 * acc)
        return np.stack(out)

    def dense(self):
        """Explicit A (n_pix x n_vox) acting on x^r; tiny inputs only."""
        def d(m):
            return m if isinstance(m, np.ndarray) else m.toarray()
        n_vox_slice = self.nx * self.ny
        A = np.zeros((self.n_pix, self.nz * n_vox_slice))
        for ks in range(self.ks):
            for kt in range(self.kt):
                if self.type == PLENOPTIC and self.nonsep:
                    S = self.scale_s3 * sum(np.kron(d(Bt), d(Bs)) * m.ravel()[None, :]
                                            for Bs, Bt, m in self.S3_2d[ks, kt])
                elif self.type == PLENOPTIC:
                    S = self.scale_s3 * np.kron(d(self.S3[1][kt]), d(self.S3[0][ks]))
                else:
                    S = None
                for n in range(self.nz):
                    B = self.scale_s1 * np.kron(d(self.S1[1][kt][n]), d(self.S1[0][ks][n]))
                    blk = B if S is None else S @ B
                    A[:, n * n_vox_slice:(n + 1) * n_vox_slice] += blk
        return A
