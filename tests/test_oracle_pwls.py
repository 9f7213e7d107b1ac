"""Pins for oracle/pwls.py (CPU only): the regulariser by direct count (golden), gains by
scalar golden-section minimisation, the gradient by central finite
differences of the profiled cost, the Hessian PSD claim and the majoriser of
Appendix A on dense tiny problems, and FISTA on toy problems."""
import json
import os

import numpy as np
import pytest
from scipy.optimize import minimize_scalar

from oracle import pwls
from oracle.system import SystemOperator
from workloads.geometry import plenoptic_camera, pose_yaw, single_camera

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def micro_problem(seed=0):
    vol = dict(nx=8, ny=8, nz=8, dx=0.8, dy=0.8, dz=0.8)
    cams = [plenoptic_camera(4, 8, 0.04, 2, 2), single_camera(32, 0.04, 2, pose=pose_yaw(30.0)),
            single_camera(32, 0.04, 2, pose=pose_yaw(-20.0))]
    ops = [SystemOperator(vol, c) for c in cams]
    rng = np.random.default_rng(seed)
    x_true = rng.random((8, 8, 8))
    g_true = [1.0, 0.7, 1.9]
    ys = [op.forward(x_true) / g for op, g in zip(ops, g_true)]
    ws = [rng.random(op.n_pix) + 0.5 for op in ops]
    return ops, ys, ws, x_true, g_true


def test_regulariser_golden():
    x = np.zeros((5, 5, 5))
    x[2, 2, 2] = 1.0
    ref = GOLDEN["regulariser"]
    assert pwls.reg_value(x, 1.0) == pytest.approx(ref["single_interior_voxel_beta1"])
    g = pwls.reg_grad(x, 1.0)
    assert g[2, 2, 2] == pytest.approx(ref["grad_centre"])
    assert g[1, 3, 2] == pytest.approx(ref["grad_neighbour"])
    assert pwls.reg_value(np.full((4, 5, 6), 3.3), 2.0) == 0.0


def test_reg_grad_finite_difference():
    rng = np.random.default_rng(1)
    x = rng.random((6, 5, 7))
    g = pwls.reg_grad(x, 0.7)
    h = 1e-6
    for idx in [(0, 0, 0), (2, 3, 4), (5, 4, 6), (3, 0, 2)]:
        e = np.zeros_like(x)
        e[idx] = h
        fd = (pwls.reg_value(x + e, 0.7) - pwls.reg_value(x - e, 0.7)) / (2 * h)
        assert g[idx] == pytest.approx(fd, rel=1e-6)


def test_gains_recovered_and_optimal():
    ops, ys, ws, x_true, g_true = micro_problem()
    st = [pwls.stats(op.forward(x_true), y, w) for op, y, w in zip(ops, ys, ws)]
    assert np.allclose(pwls.gains(st), g_true, rtol=1e-12)
    rng = np.random.default_rng(3)
    x = rng.random((8, 8, 8))
    Ax = [op.forward(x) for op in ops]
    gam = pwls.gains([pwls.stats(a, y, w) for a, y, w in zip(Ax, ys, ws)])
    for c in (1, 2):
        f = lambda g: 0.5 * np.sum(ws[c] * (Ax[c] - g * ys[c]) ** 2)
        res = minimize_scalar(f, bracket=(0.0, 5.0), method="golden", tol=1e-12)
        assert gam[c] == pytest.approx(res.x, rel=1e-7)


def test_profiled_gradient_finite_difference():
    ops, ys, ws, _, _ = micro_problem()
    rng = np.random.default_rng(4)
    x = rng.random((8, 8, 8))
    beta, nu = 0.05, 0.01
    g = pwls.gradient(x, ops, ys, ws, beta, nu)
    h = 1e-5
    for idx in [(0, 0, 0), (3, 4, 5), (7, 7, 7), (2, 6, 1)]:
        e = np.zeros_like(x)
        e[idx] = h
        fd = (pwls.profiled_cost(x + e, ops, ys, ws, beta, nu) - pwls.profiled_cost(x - e, ops, ys, ws, beta, nu)) / (2 * h)
        assert g[idx] == pytest.approx(fd, rel=1e-6, abs=1e-9 * np.abs(g).max())


def _reg_hessian(shape, beta):
    n = int(np.prod(shape))
    Hm = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        Hm[:, j] = pwls.reg_grad(e.reshape(shape), beta).ravel()
    return Hm


def test_hessian_psd_and_majoriser():
    """Appendix A: H = A1'A1 + hess R + sum A_c' G_c^2 A_c >= 0 and <= D + c_R beta I."""
    ops, ys, ws, _, _ = micro_problem()
    beta = 0.3
    A = [np.sqrt(w)[:, None] * op.dense() for op, w in zip(ops, ws)]
    yt = [np.sqrt(w) * y for y, w in zip(ys, ws)]
    HR = _reg_hessian((8, 8, 8), beta)
    Hm = A[0].T @ A[0] + HR
    for Ac, y in zip(A[1:], yt[1:]):
        G = np.eye(len(y)) - np.outer(y, y) / (y @ y)
        Hm += Ac.T @ G @ G @ Ac
    ev = np.linalg.eigvalsh(Hm)
    assert ev.min() >= -1e-12 * ev.max()
    d = pwls.majoriser(ops, ws, beta, (8, 8, 8)).ravel()
    M = np.diag(d) - Hm
    assert np.linalg.eigvalsh(M).min() >= -1e-9 * ev.max()
    # profiled Hessian equals the finite-difference Jacobian of the profiled gradient
    rng = np.random.default_rng(9)
    x, v = rng.random((8, 8, 8)), rng.normal(size=(8, 8, 8))
    h = 1e-4
    fd = (pwls.gradient(x + h * v, ops, ys, ws, beta, 0.0) - pwls.gradient(x - h * v, ops, ys, ws, beta, 0.0)) / (2 * h)
    # (the profiled Hessian at x is not exactly the G_c form away from optimum gains; check the PSD form's
    # quadratic action against the FD curvature only in sign)
    assert v.ravel() @ fd.ravel() >= 0.0


def test_paper_26beta_fails_under_literal_regulariser():
    """Reading Z16: lambda_max(hess R)/beta exceeds 26 already on a 3^3 grid (27) -> constant 36."""
    lam3 = np.linalg.eigvalsh(_reg_hessian((3, 3, 3), 1.0)).max()
    lam6 = np.linalg.eigvalsh(_reg_hessian((6, 6, 6), 1.0)).max()
    assert lam3 == pytest.approx(27.0, abs=1e-9)
    assert 26.0 < lam6 <= pwls.MAJORISER_C


class _Identity:
    def __init__(self, n):
        self.n_vox = self.n_pix = n

    def forward(self, x):
        return np.asarray(x, np.float64).ravel()

    def adjoint(self, y):
        return np.asarray(y, np.float64).ravel()


def test_fista_identity_toy():
    op = _Identity(1)
    x = pwls.fista([op], [np.array([3.0])], [np.array([1.0])], 0.0, 0.0, (1, 1, 1), 50)
    assert x.ravel()[0] == pytest.approx(3.0, abs=1e-6)
    x = pwls.fista([op], [np.array([3.0])], [np.array([1.0])], 0.0, 0.4, (1, 1, 1), 50)
    assert x.ravel()[0] == pytest.approx(2.6, abs=1e-6)       # soft threshold by nu


def test_fista_decreases_cost_and_stays_nonnegative():
    ops, ys, ws, x_true, _ = micro_problem()
    beta, nu = 1e-3, 0.0
    costs = []
    cb = lambda it, x: costs.append(pwls.profiled_cost(x, ops, ys, ws, beta, nu))
    x = pwls.fista(ops, ys, ws, beta, nu, (8, 8, 8), 30, callback=cb)
    assert (x >= 0).all()
    assert costs[-1] < 0.1 * costs[0]
