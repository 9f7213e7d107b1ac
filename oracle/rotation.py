"""Three-pass shear rotation of the voxel volume (paper §3.1).

p = Theta p^r, Theta = D_Theta S_z S_x S_y (eqn,rot,decomp P:1127-1135),
with unit shears  S_y: y' = a_yx x + y + a_yz z;  S_x: x' = x + a_xy y + a_xz z;
S_z: z' = a_zx x + a_zy y + z.  The paper gives no closed form; the one below
 solves the 9 entry equations row by row (pinned in tests by
re-multiplying the factors, and by rotating a smooth blob against the analytic
rotation).

D_Theta only relabels the voxel sizes: Delta^r = Delta / D.  Each shear
is an L2 projection onto the same grid, x^r = E^y E^x E^z x, with
block-Toeplitz E (eqn,rot,toeplitz P:1186-1195).  Derived here for E^z (the other
passes permute the axes):

  [E^z]_ij = 1/(Dx Dy Dz) * integral over the (x,y) cell of i of
             Lambda_Dz(z_j - z_i - a_zx x - a_zy y) dx dy,   Lambda_D(t) = max(0, D - |t|)
           = (1/Dz) (Lambda_Dz * U_{|a_zx| Dx} * U_{|a_zy| Dy})(z_j - z_i - sigma_i),
  sigma_i = a_zx x_i + a_zy y_i,  U_w = uniform density of width w (delta if w = 0).

(1/Dz) Lambda * U is the paper's "piecewise quadratic" g^z integrated over the source
cell.  Every pass keeps the grid dims with zeros outside (crop, Z14).

Poses beyond 45 degrees (NEXT-4): Theta = P Theta' with P the closest of the 24 cube
rotations (reading R7); P is applied first as an exact index relabelling x_P(q) = x(P q), then the
three shears of Theta'.
"""
import numpy as np
import scipy.sparse as sp


class NotDecomposable(ValueError):
    pass


def decompose(R):
    """Closed-form D, shear coefficients of Theta = R (row-major 9-tuple)."""
    (Txx, Txy, Txz, Tyx, Tyy, Tyz, Tzx, Tzy, Tzz) = [float(v) for v in R]
    Dy = Tyy
    if abs(Dy) < 1e-6:
        raise NotDecomposable("D_y ~ 0 (rotation >= 45 deg needs a quarter-turn permutation)")
    a_yx = Tyx / Dy
    a_yz = Tyz / Dy
    Dx = Txx - Txy * a_yx
    if abs(Dx) < 1e-6:
        raise NotDecomposable("D_x ~ 0")
    a_xy = Txy / Dx
    a_xz = Txz / Dx - a_xy * a_yz
    m_xx = 1.0 + a_xy * a_yx
    m_xz = a_xz + a_xy * a_yz
    alpha = Tzx - a_yx * Tzy
    beta = m_xx * Tzy - a_xy * Tzx
    Dz = Tzz - alpha * m_xz - beta * a_yz
    if abs(Dz) < 1e-6:
        raise NotDecomposable("D_z ~ 0")
    a_zx = alpha / Dz
    a_zy = beta / Dz
    return dict(D=(Dx, Dy, Dz), a_yx=a_yx, a_yz=a_yz, a_xy=a_xy, a_xz=a_xz, a_zx=a_zx, a_zy=a_zy)


def factor_matrices(dec):
    Dx, Dy, Dz = dec["D"]
    D = np.diag([Dx, Dy, Dz])
    Sy = np.array([[1, 0, 0], [dec["a_yx"], 1, dec["a_yz"]], [0, 0, 1]], float)
    Sx = np.array([[1, dec["a_xy"], dec["a_xz"]], [0, 1, 0], [0, 0, 1]], float)
    Sz = np.array([[1, 0, 0], [0, 1, 0], [dec["a_zx"], dec["a_zy"], 1]], float)
    return D, Sz, Sx, Sy


# ---- the 1D shear kernel: (1/D) (Lambda_D * U_wa * U_wb)(d), exact piecewise polynomial ----

def _lam1(t, D):
    """int_{-inf}^t Lambda_D."""
    return np.where(t <= -D, 0.0, np.where(t <= 0.0, 0.5 * (t + D) ** 2,
                    np.where(t < D, D * D - 0.5 * (D - t) ** 2, D * D)))


def _lam2(t, D):
    """Second antiderivative of Lambda_D."""
    return np.where(t <= -D, 0.0, np.where(t <= 0.0, (t + D) ** 3 / 6.0,
                    np.where(t < D, D * D * t + (D - t) ** 3 / 6.0, D * D * t)))


def shear_kernel(d, D, wa, wb):
    """Weight of a source cell at offset d (= z_j - z_i - sigma_i) for cell size D."""
    d = np.asarray(d, np.float64)
    tiny = 1e-9 * D
    ws = sorted([w for w in (abs(wa), abs(wb)) if w > tiny])
    if not ws:
        return np.maximum(0.0, D - np.abs(d)) / D
    if len(ws) == 1:
        w = ws[0]
        return (_lam1(d + 0.5 * w, D) - _lam1(d - 0.5 * w, D)) / (w * D)
    wa, wb = ws
    return (_lam2(d + 0.5 * (wa + wb), D) - _lam2(d + 0.5 * (wb - wa), D)
            - _lam2(d - 0.5 * (wb - wa), D) + _lam2(d - 0.5 * (wa + wb), D)) / (wa * wb * D)


def _centres(n, d):
    return (np.arange(n, dtype=np.float64) - (n - 1) * 0.5) * d


def shear_matrix(dims, vox, axis, c1, c2):
    """Sparse E for one pass on a (nx, ny, nz) grid with voxel sizes vox (x fastest).

    axis 'z': lines along z, sigma = c1*x + c2*y  (c1, c2) = (a_zx, a_zy)
    axis 'x': lines along x, sigma = c1*y + c2*z  (c1, c2) = (a_xy, a_xz)
    axis 'y': lines along y, sigma = c1*x + c2*z  (c1, c2) = (a_yx, a_yz)
    """
    nx, ny, nz = dims
    dx, dy, dz = vox
    X, Y, Z = np.meshgrid(_centres(nx, dx), _centres(ny, dy), _centres(nz, dz), indexing="ij")
    IX, IY, IZ = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    if axis == "z":
        D, sig, wa, wb, pos, n = dz, c1 * X + c2 * Y, c1 * dx, c2 * dy, IZ, nz
    elif axis == "x":
        D, sig, wa, wb, pos, n = dx, c1 * Y + c2 * Z, c1 * dy, c2 * dz, IX, nx
    elif axis == "y":
        D, sig, wa, wb, pos, n = dy, c1 * X + c2 * Z, c1 * dx, c2 * dz, IY, ny
    else:
        raise ValueError(axis)
    reach = D + 0.5 * (abs(wa) + abs(wb))
    mmax = int(np.ceil((np.abs(sig).max() + reach) / D)) + 1
    flat = (IX + nx * (IY + ny * IZ)).ravel()
    rows, cols, vals = [], [], []
    for m in range(-mmax, mmax + 1):
        jpos = pos + m
        ok = (jpos >= 0) & (jpos < n)
        w = shear_kernel(m * D - sig, D, wa, wb)
        ok &= w > 0.0
        if axis == "z":
            jflat = IX + nx * (IY + ny * jpos)
        elif axis == "x":
            jflat = jpos + nx * (IY + ny * IZ)
        else:
            jflat = IX + nx * (jpos + ny * IZ)
        rows.append(flat[ok.ravel()])
        cols.append(jflat.ravel()[ok.ravel()])
        vals.append(w.ravel()[ok.ravel()])
    N = nx * ny * nz
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))


def _proper_signed_permutations():
    """The 24 rotations of the cube (signed permutation matrices with det +1), identity first."""
    import itertools
    out = [np.eye(3)]
    for perm in itertools.permutations(range(3)):
        for signs in itertools.product((1.0, -1.0), repeat=3):
            P = np.zeros((3, 3))
            for r in range(3):
                P[r, perm[r]] = signs[r]
            if np.linalg.det(P) > 0.5 and not np.array_equal(P, np.eye(3)):
                out.append(P)
    return out


def quarter_turn(R):
    """NEXT-4 reading R7: Theta = P Theta' with P the cube rotation closest to Theta (largest trace of
    P^T Theta; ties keep the earlier candidate, identity first), so the residual Theta' is within the
    range the three-shear decomposition handles (P:1117-1119 restrict the decomposition to < 45 deg)."""
    T = np.asarray(R, np.float64).reshape(3, 3)
    best, bestv = None, -np.inf
    for P in _proper_signed_permutations():
        v = np.trace(P.T @ T)
        if v > bestv + 1e-12:
            best, bestv = P, v
    return best, best.T @ T


def permutation_matrix(P, dims, vox):
    """Sparse relabelling x_P(q) = x(P q) on a grid symmetric about the origin (exact for a signed
    permutation when the permuted axes have equal cell counts and sizes)."""
    nx, ny, nz = dims
    n = (nx, ny, nz)
    for b in range(3):
        a = int(np.argmax(np.abs(P[b])))
        if n[a] != n[b] or abs(vox[a] - vox[b]) > 1e-12 * vox[b]:
            raise NotDecomposable("quarter-turn permutation needs equal dims and voxel sizes on the permuted axes")
    I = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    src = np.zeros_like(I)
    for b in range(3):
        a = int(np.argmax(np.abs(P[b])))
        src[:, b] = I[:, a] if P[b, a] > 0 else n[b] - 1 - I[:, a]
    rows = I[:, 0] + nx * (I[:, 1] + ny * I[:, 2])
    cols = src[:, 0] + nx * (src[:, 1] + ny * src[:, 2])
    N = nx * ny * nz
    return sp.csr_matrix((np.ones(N), (rows, cols)), shape=(N, N))


class Rotation:
    """x^r = E^y E^x E^z P_perm x on the relabelled grid (voxel sizes Delta/D); P_perm is the exact
    quarter-turn relabelling of reading R7 (identity for poses within 45 degrees)."""

    def __init__(self, R, dims, vox):
        self.P, Tres = quarter_turn(R)
        self.Pm = None if np.array_equal(self.P, np.eye(3)) else permutation_matrix(self.P, dims, vox)
        self.dec = decompose(Tres.ravel())
        D = self.dec["D"]
        self.dims = dims
        self.vox_r = (vox[0] / D[0], vox[1] / D[1], vox[2] / D[2])
        d = self.dec
        self.Ez = shear_matrix(dims, self.vox_r, "z", d["a_zx"], d["a_zy"])
        self.Ex = shear_matrix(dims, self.vox_r, "x", d["a_xy"], d["a_xz"])
        self.Ey = shear_matrix(dims, self.vox_r, "y", d["a_yx"], d["a_yz"])

    def forward(self, x):
        v = np.asarray(x, np.float64).ravel()
        if self.Pm is not None:
            v = self.Pm @ v
        return (self.Ey @ (self.Ex @ (self.Ez @ v))).reshape(self.dims[2], self.dims[1], self.dims[0])

    def adjoint(self, xr):
        v = np.asarray(xr, np.float64).ravel()
        v = self.Ez.T @ (self.Ex.T @ (self.Ey.T @ v))
        if self.Pm is not None:
            v = self.Pm.T @ v
        return v.reshape(self.dims[2], self.dims[1], self.dims[0])

    def dense(self):
        M = self.Ey @ self.Ex @ self.Ez
        if self.Pm is not None:
            M = M @ self.Pm
        return M.toarray()
