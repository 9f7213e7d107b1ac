"""Pins for the view-subset gradient of oracle/pwls.py (sec,subset P:360-388, reading Z19/R5), CPU only.

* partition: the n_subsets subsets are disjoint, cover all K views, and S_m = {k : k mod M = m} with
  k = k_t K_s + k_s (every M-th view of the lexicographically ordered angular plane);
* one subset (M = 1) reproduces the exact profiled gradient;
* unbiasedness of the scaled subset sums (the reason for the K/|S| factor): for equal-size subsets the mean
  over m of (K/|S_m|) A_{S_m} x equals A x and of (K/|S_m|) A_{S_m}^T r equals A^T r;
* the subset gradient equals a direct evaluation of eqn,subset written with explicit per-view operators
  (each A_ck assembled from the oracle with a one-view list), so a dropped scale, a swapped gain or a
  wrong subset fails.
"""
import numpy as np
import pytest

from oracle import pwls
from oracle.system import build_system
from workloads import make_config, normal_vector, uniform_vector, uniform_volume


@pytest.mark.parametrize("ks,kt,M", [(2, 2, 2), (4, 4, 4), (4, 4, 3), (8, 8, 5), (3, 2, 6)])
def test_partition(ks, kt, M):
    seen = []
    for m in range(M):
        S = pwls.subset_views(ks, kt, M, m)
        for (a, b) in S:
            k = b * ks + a
            assert k % M == m
            seen.append(k)
    assert sorted(seen) == list(range(ks * kt))


def _data(name):
    cfg = make_config(name)
    ops = build_system(cfg)
    x = uniform_volume(cfg["volume"], 0).astype(np.float64)
    ys = [uniform_vector(op.n_pix, 1 + c).astype(np.float64) for c, op in enumerate(ops)]
    ws = [(0.5 + uniform_vector(op.n_pix, 5 + c)).astype(np.float64) for c, op in enumerate(ops)]
    return cfg, ops, x, ys, ws


def test_one_subset_is_exact():
    cfg, ops, x, ys, ws = _data("tiny_multi")
    g1 = pwls.gradient_subset(x, ops, ys, ws, 0.01, 0.1, 1, 0)
    g = pwls.gradient(x, ops, ys, ws, 0.01, 0.1)
    assert np.abs(g1 - g).max() <= 1e-12 * np.abs(g).max()


@pytest.mark.parametrize("M", [2, 4])
def test_scaled_subset_sums_are_unbiased(M):
    cfg, ops, x, ys, ws = _data("tiny_k4")
    op = ops[0]
    K = op.n_views
    r = normal_vector(op.n_pix, 3).astype(np.float64)
    fx = np.zeros(op.n_pix)
    bt = np.zeros(op.n_vox)
    for m in range(M):
        S = pwls.subset_views(op.camera.ks, op.camera.kt, M, m)
        fx += K / len(S) * op.forward(x, S) / M
        bt += K / len(S) * op.adjoint(r, S) / M
    ref_f, ref_b = op.forward(x), op.adjoint(r)
    assert np.abs(fx - ref_f).max() <= 1e-12 * np.abs(ref_f).max()
    assert np.abs(bt - ref_b).max() <= 1e-12 * np.abs(ref_b).max()


@pytest.mark.parametrize("M,m", [(2, 1), (3, 2), (4, 0)])
def test_subset_gradient_matches_direct_evaluation(M, m):
    cfg, ops, x, ys, ws = _data("tiny_multi")
    beta, nu = 0.02, 0.05
    got = pwls.gradient_subset(x, ops, ys, ws, beta, nu, M, m)
    # direct: per-view operators, then the formula of eqn,subset with reading Z19
    yhat, scales, views = [], [], []
    for op in ops:
        ks, kt = op.camera.ks, op.camera.kt
        S = [(k % ks, k // ks) for k in range(ks * kt) if k % M == m]
        s = ks * kt / len(S)
        yhat.append(s * sum(op.forward(x, [v]) for v in S))
        scales.append(s)
        views.append(S)
    gam = [1.0] + [float(np.sum(w * y * a) / np.sum(w * y * y)) for a, y, w in zip(yhat[1:], ys[1:], ws[1:])]
    ref = np.zeros(x.size)
    for op, a, y, w, gc, s, S in zip(ops, yhat, ys, ws, gam, scales, views):
        res = w * (a - gc * y)
        ref += s * sum(op.adjoint(res, [v]) for v in S)
    ref = ref.reshape(x.shape) + pwls.reg_grad(x, beta) + nu
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_subset_fista_decreases_cost():
    cfg = make_config("tiny_k4")
    ops = build_system(cfg)
    from workloads import flame_volume
    xt = flame_volume(cfg["volume"]).astype(np.float64)
    ys = [op.forward(xt) for op in ops]
    ws = [np.ones(op.n_pix) for op in ops]
    shape = xt.shape
    c0 = pwls.profiled_cost(np.zeros(shape), ops, ys, ws, 0.0, 0.0)
    x = pwls.fista(ops, ys, ws, 0.0, 0.0, shape, 8, n_subsets=4)
    assert pwls.profiled_cost(x, ops, ys, ws, 0.0, 0.0) < 0.2 * c0
