"""Pins for the two oracle parts SURVEY §8(c)-C9 left "parity unpinned" (What's weak 1).
CPU only; each expected value is derived here by hand from the paper's definitions, not from the oracle.

1. Absolute scale of y (reading Z7: the literal building blocks f^p = B f^q / V^p, and
   y = sqrt(V^d) sum_k f^d_k).  An "identity-plane" single-lens camera -- one slice exactly in focus on the
   detector (1/z + 1/D = 1/f), detector pitch = |lambda| x voxel pitch, one angular cell (K = 1) -- has
   B^{dq}/V^d = I per axis up to the image inversion (the identity special case of eqn,xport,ip), so
   the composed model must give  y = sqrt(V^d) * Dz * x  (x flipped in s and t), with V^d = prod_axes
   Dp D0/|b_d| (reading Z6).  Dropping the 1/V^d of P:835 (the P:989 variant) or the sqrt(V^d) of P:956 changes
   y by V^d or sqrt(V^d) = 0.008 / 6.4e-5, which this test rejects.
2. FISTA momentum (tab,alg missing, reading Z18; P:341-349 names FISTA of Beck & Teboulle):
   (a) the first three iterates of a 2-variable problem worked out by hand (momentum (t_k - 1)/t_{k+1} with
       t_{k+1} = (1 + sqrt(1 + 4 t_k^2))/2, t_0 = 1); ISTA or another momentum gives a different x_3;
   (b) Beck & Teboulle's rate F(x_k) - F* <= 2 ||x_0 - x*||_D^2 / (k+1)^2 (their Thm 4.4 in the D-metric of a
       diagonal majoriser D >= H) on an ill-conditioned quadratic, which plain projected gradient (ISTA, the
       same steps without momentum) violates on the same problem.
"""
import math

import numpy as np
import pytest

from oracle import pwls
from oracle.system import SystemOperator


# ----------------------------------------------------------------------------------------------- 1. scale of y
def test_single_lens_identity_plane_scale():
    f, z, D = 50.0, 300.0, 60.0            # 1/300 + 1/60 = 1/50: the slice plane is in focus on the detector
    dp = 0.04                              # detector pitch
    dx = dp * z / D                        # voxel pitch = dp / |lambda|, lambda = -D/z (magnification)
    n = 16
    vol = dict(nx=n, ny=n, nz=1, dx=dx, dy=dx, dz=dx)
    ap = 12.0                              # K = 1: one angular cell D0 = the whole aperture
    cam = dict(type=0, basis=0, f_main=f, ap_s=ap, ap_t=ap, d_scene=z, k_s=1, k_t=1, d_det=D, d_mu_m=0.0,
               d_d_mu=0.0, f_mu=0.0, fill=0.0, nl_s=0, nl_t=0, n_a=0, n_s=n, n_t=n, px_s=dp, px_t=dp,
               R=(1.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0))
    op = SystemOperator(vol, cam)
    x = np.random.default_rng(5).random((1, n, n))
    y = op.forward(x).reshape(n, n)
    v_axis = dp * ap / D                   # V^d per axis = Dp D0 / |b_d|, X^{0d} = T_{-D} (reading Z6)
    expect = math.sqrt(v_axis * v_axis) * dx * x[0, ::-1, ::-1]
    assert np.abs(y - expect).max() <= 1e-12 * np.abs(expect).max()
    # and the adjoint (literal transpose) carries the same scalar
    g = op.adjoint(y.ravel()).reshape(1, n, n)
    assert np.abs(g - (v_axis * dx) ** 2 * x).max() <= 1e-12 * np.abs(g).max()


# ----------------------------------------------------------------------------------------------- 2. FISTA
class _Matrix:
    """One 'camera' whose forward is a matrix (W = 1, gain 1: F(x) = 1/2 ||A x - y||^2 + R(x) with beta = 0)."""

    def __init__(self, A):
        self.A = np.asarray(A, np.float64)
        self.n_pix, self.n_vox = self.A.shape

    def forward(self, x):
        return self.A @ np.asarray(x, np.float64).ravel()

    def adjoint(self, y):
        return self.A.T @ np.asarray(y, np.float64).ravel()


def test_fista_hand_iterates_two_variables():
    # A^T A = H = [[2, 1], [1, 2]], A^T y = b = [3, 2], majoriser d = H 1 = [3, 3], x* = H^-1 b = [4/3, 1/3] > 0
    A = np.array([[1.0, 1.0], [1.0, 0.0], [0.0, 1.0]])
    y = np.array([1.0, 2.0, 1.0])
    op = _Matrix(A)
    xs = []
    pwls.fista([op], [y], [np.ones(3)], 0.0, 0.0, (2, 1, 1), 3, callback=lambda it, x: xs.append(x.ravel().copy()))
    assert np.allclose(pwls.majoriser([op], [np.ones(3)], 0.0, (2, 1, 1)).ravel(), [3.0, 3.0], rtol=0, atol=1e-15)
    # by hand: z0 = x0 = 0, grad = H z - b
    #   x1 = z0 - (H z0 - b)/3 = [1, 2/3];       t1 = (1 + sqrt 5)/2,  z1 = x1 + (t0 - 1)/t1 (x1 - x0) = x1
    #   x2 = z1 - (H z1 - b)/3 = [10/9, 5/9];    t2 = (1 + sqrt(1 + 4 t1^2))/2,  m = (t1 - 1)/t2
    #   z2 = x2 + m (x2 - x1) = [10/9 + m/9, 5/9 - m/9];  H z2 - b = (m - 2)/9 [1, -1]
    #   x3 = z2 - (H z2 - b)/3 = [10/9 + m/9 - (m - 2)/27, 5/9 - m/9 + (m - 2)/27]
    t1 = (1.0 + math.sqrt(5.0)) / 2.0
    t2 = (1.0 + math.sqrt(1.0 + 4.0 * t1 * t1)) / 2.0
    m = (t1 - 1.0) / t2
    hand = [np.array([1.0, 2.0 / 3.0]), np.array([10.0 / 9.0, 5.0 / 9.0]),
            np.array([10.0 / 9.0 + m / 9.0 - (m - 2.0) / 27.0, 5.0 / 9.0 - m / 9.0 + (m - 2.0) / 27.0])]
    for got, exp in zip(xs, hand):
        assert np.abs(got - exp).max() <= 1e-14
    # what the pin rejects: ISTA (m = 0) and the common slips (t_k - 1)/t_k, t_k / t_{k+1}, t_{k+1} = t_k + 1
    for wrong in (0.0, (t1 - 1.0) / t1, t1 / t2, 1.0 / 3.0):
        x3w = np.array([10.0 / 9.0 + wrong / 9.0 - (wrong - 2.0) / 27.0, 5.0 / 9.0 - wrong / 9.0 + (wrong - 2.0) / 27.0])
        assert np.abs(x3w - xs[2]).max() > 1e-3


def _ill_conditioned(n=40):
    # A = lower bidiagonal blur (1 on the diagonal and sub-diagonal): H = A^T A has eigenvalues 2 + 2 cos(theta),
    # condition number ~ 4 (n + 1)^2 / pi^2, the slowest mode the alternating one; x* > 0 (the constraint x >= 0
    # is inactive) with a large component along that slow mode
    A = np.eye(n + 1, n) + np.eye(n + 1, n, -1)
    i = np.arange(n)
    x_star = 1.0 + 0.5 * (-1.0) ** i * np.sin(np.pi * (i + 1) / (n + 1))
    return A, A @ x_star, x_star


def test_fista_beck_teboulle_rate():
    A, y, x_star = _ill_conditioned()
    n = x_star.size
    op = _Matrix(A)
    w = [np.ones(A.shape[0])]
    d = pwls.majoriser([op], w, 0.0, (n, 1, 1)).ravel()
    H = A.T @ A
    assert np.linalg.eigvalsh(np.diag(d) - H).min() >= -1e-12      # D majorises H (De Pierro)
    F = lambda x: 0.5 * np.sum((A @ x - y) ** 2)
    bound0 = 2.0 * np.sum(d * x_star ** 2)                        # 2 ||x0 - x*||_D^2, x0 = 0
    iters = 1500
    gaps = []
    pwls.fista([op], [y], w, 0.0, 0.0, (n, 1, 1), iters, callback=lambda it, x: gaps.append(F(x.ravel())))
    k = np.arange(1, iters + 1)
    assert np.all(np.array(gaps) <= bound0 / (k + 1.0) ** 2 * (1 + 1e-9) + 1e-12)
    # the same steps without momentum (ISTA) break the bound on this problem: the bound has teeth
    x = np.zeros(n)
    viol = False
    for kk in range(1, iters + 1):
        x = np.maximum(0.0, x - (H @ x - A.T @ y) / d)
        viol |= F(x) > bound0 / (kk + 1.0) ** 2
    assert viol
