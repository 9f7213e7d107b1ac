"""Light transport between two planes, one separable axis (paper §2.3).

Coefficients on plane p follow from the L2 projection eqn,xport:
f^p_k = (1/V^p) B^{pq}_k f^q_k, with B^{pq}_k = B_{k,s} (x) B_{k,t}
(eqn,xport,sep P:904-910).  One 1D factor entry is the (s,u) inner product of
eqn,xport,ip:

  [B]_ij = << b((X^pq_s(s,u) - s_i)/Dp) a((X^0q_s(s,u) - s_k)/D0), b((s - s_j)/Dq) >>

The tables that close eqn,xport,int (tab,dirac / tab,pillbox) are
missing; the closed form used here (reading Z5) follows from
substituting u -> s_0 = X^0q_s(s,u) (du = ds_0/|b_q|):

  s_p = lam*s + mu*s_0 + nu,   lam = P - Q a_q/b_q,  mu = Q/b_q,  nu = o_pq - Q o_q/b_q
  c_i = (s_i - nu - mu s_k)/lam           (row-i kernel centre on the source plane)
  pillbox: W = (D0|mu| + Dp)/(2|lam|),  w = |D0|mu| - Dp|/(2|lam|),  H = min(D0, Dp/|mu|)
  Dirac:   W = w = Dp/(2|lam|),  H = D0
  Trap(x) = H on |x|<=w, linear to 0 at |x|=W
  [B]_ij = (1/|b_q|) * integral over source cell j of Trap(s - c_i) ds

In the paper's notation: alpha = 1/lam, tau = (shift, W, w), h*g = Trap/|b_q|.
This closed form is pinned in tests against an exact polygon-area evaluation of the
inner product itself, not against itself.

V^p = Dp * D0 / |b_p| per axis (b_p = X^0p_su); for the Dirac basis the
same value is used (reading Z6: one angular factor, identity transport exact).
"""
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .optics import Affine1D, compose, invert

PILLBOX, DIRAC = 0, 1


@dataclass(frozen=True)
class Plane:
    """One axis of an optical plane: n cells of width `delta` centred on c0, and X^{0p}."""
    n: int
    delta: float
    X0: Affine1D
    c0: float = 0.0

    def centres(self):
        # s_i = c0 + (i - (n-1)/2) * delta
        i = np.arange(self.n, dtype=np.float64)
        return self.c0 + (i - (self.n - 1) * 0.5) * self.delta


class DegenerateGeometry(ValueError):
    pass


def ray_coefficients(src, dst):
    """(lam, mu, nu) with s_dst = lam*s_src + mu*s_0 + nu for a ray through s_src and s_0."""
    Xpq = compose(invert(dst.X0), src.X0)          # X^{pq} = (X^{0p})^{-1} o X^{0q}
    P, Q, o_pq = Xpq.m00, Xpq.m01, Xpq.o0
    a_q, b_q, o_q = src.X0.m00, src.X0.m01, src.X0.o0
    if b_q == 0.0:
        raise DegenerateGeometry("source plane coincides with the angular plane (b_q = 0)")
    lam = P - Q * a_q / b_q
    mu = Q / b_q
    nu = o_pq - Q * o_q / b_q
    if lam == 0.0:
        raise DegenerateGeometry("destination conjugate to the angular plane (lambda = 0)")
    return lam, mu, nu


def trapezoid(lam, mu, dp, d0, basis):
    """(W, w, H) of the blur kernel on the source plane (closes the missing tables)."""
    al = abs(lam)
    if basis == DIRAC:
        return dp / (2.0 * al), dp / (2.0 * al), d0
    am = abs(mu)
    W = (d0 * am + dp) / (2.0 * al)
    w = abs(d0 * am - dp) / (2.0 * al)
    H = d0 if am == 0.0 else min(d0, dp / am)
    return W, w, H


def trap_value(x, W, w, H):
    ax = np.abs(x)
    ramp = H * (W - ax) / (W - w) if W > w else np.zeros_like(ax)
    return np.where(ax <= w, H, np.where(ax < W, ramp, 0.0))


def trap_integral(lo, hi, W, w, H):
    """Exact integral of Trap over [lo, hi] (arrays): midpoint rule on each linear piece."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    total = np.zeros(np.broadcast(lo, hi).shape)
    for p0, p1 in ((-W, -w), (-w, w), (w, W)):
        if p1 <= p0:
            continue
        l = np.maximum(lo, p0)
        h = np.minimum(hi, p1)
        m = h > l
        mid = np.where(m, 0.5 * (l + h), 0.0)
        total += np.where(m, (h - l) * trap_value(mid, W, w, H), 0.0)
    return total


def row_params(src, dst, s_k, d0, basis):
    """Per destination row i: kernel centre c_i on the source plane, plus (W, w, H)."""
    lam, mu, nu = ray_coefficients(src, dst)
    W, w, H = trapezoid(lam, mu, dst.delta, d0, basis)
    c = (dst.centres() - nu - mu * s_k) / lam
    return c, W, w, H


def band(src, dst, s_k, d0, basis):
    """Analytic band [j_lo, j_hi] per row (reading Z21: open support; -1/-2 style empty = lo>hi).

    j in band(i) iff s_j + Dq/2 > c_i - W and s_j - Dq/2 < c_i + W, evaluated as
    j_lo = floor((c_i - W - s_0 - Dq/2)/Dq) + 1, j_hi = ceil((c_i + W - s_0 + Dq/2)/Dq) - 1,
    clamped to [0, n_src - 1], where s_0 is the first source cell centre.
    """
    c, W, w, H = row_params(src, dst, s_k, d0, basis)
    dq = src.delta
    s0 = src.c0 + (0.0 - (src.n - 1) * 0.5) * dq
    lo = np.floor((c - W - s0 - 0.5 * dq) / dq) + 1.0
    hi = np.ceil((c + W - s0 + 0.5 * dq) / dq) - 1.0
    lo = np.maximum(lo, 0.0)
    hi = np.minimum(hi, float(src.n - 1))
    empty = hi < lo
    lo = np.where(empty, 0.0, lo).astype(np.int64)
    hi = np.where(empty, -1.0, hi).astype(np.int64)
    return lo, hi


def entries(src, dst, s_k, d0, basis, rows, cols):
    """[B^{pq}_k]_{rows, cols} (broadcast arrays of indices) in fp64, closed form."""
    c, W, w, H = row_params(src, dst, s_k, d0, basis)
    sj = src.centres()[cols]
    ci = c[rows]
    bq = abs(src.X0.m01)
    return trap_integral(sj - 0.5 * src.delta - ci, sj + 0.5 * src.delta - ci, W, w, H) / bq


def transport_dense(src, dst, s_k, d0, basis):
    """Every entry of the 1D factor (n_dst x n_src), no band logic: the tiny-input definition."""
    rows, cols = np.meshgrid(np.arange(dst.n), np.arange(src.n), indexing="ij")
    return entries(src, dst, s_k, d0, basis, rows, cols)


def transport_sparse(src, dst, s_k, d0, basis, margin=1):
    """Same matrix as CSR, evaluating only the analytic band widened by `margin` cells."""
    lo, hi = band(src, dst, s_k, d0, basis)
    rows, cols = [], []
    for i in range(dst.n):
        if hi[i] < lo[i]:
            continue
        j = np.arange(max(lo[i] - margin, 0), min(hi[i] + margin, src.n - 1) + 1)
        rows.append(np.full(j.shape, i))
        cols.append(j)
    if not rows:
        return sp.csr_matrix((dst.n, src.n))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = entries(src, dst, s_k, d0, basis, rows, cols)
    keep = vals != 0.0
    return sp.csr_matrix((vals[keep], (rows[keep], cols[keep])), shape=(dst.n, src.n))


def basis_volume(plane, d0):
    """V^p per axis: ||a(X^0p_s/D0) b(s/Dp)||^2 = Dp * D0 / |X^0p_su|."""
    return plane.delta * d0 / abs(plane.X0.m01)


def angular_centres(k, d0):
    """Angular sample centres s_k = (k - (K-1)/2) D0 tiling a square aperture (reading Z4)."""
    return (np.arange(k, dtype=np.float64) - (k - 1) * 0.5) * d0
