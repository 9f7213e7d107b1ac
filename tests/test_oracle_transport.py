"""Pins for oracle/optics.py and oracle/transport.py (CPU only).

Each test checks the oracle against something other than itself: ray-transfer
arithmetic, the exact polygon area of the paper's inner product (eqn,xport,ip
P:851-875), the p,q symmetry the paper states, the identity transport,
parallelogram row mass, the tensor tiling of the angular plane, and Kronecker
separability (eqn,xport,sep P:904-910).
"""
import math

import numpy as np
import pytest

from oracle.optics import Affine1D, compose, invert, lens, translate
from oracle.transport import (DIRAC, PILLBOX, DegenerateGeometry, Plane, band, basis_volume, entries,
                              ray_coefficients, row_params, transport_dense, transport_sparse)
from tests.brute import interval_overlap, strip_polygon_area

F = 50.0


def H(a):
    """Homogeneous 3x3 matrix of an Affine1D (test-side, numpy linear algebra)."""
    return np.array([[a.m00, a.m01, a.o0], [a.m10, a.m11, a.o1], [0.0, 0.0, 1.0]])


# ---------------------------------------------------------------- optics
def test_translation_examples():
    s, u = translate(60.0).apply(1.0, 0.1)
    assert (s, u) == pytest.approx((7.0, 0.1))
    assert compose(translate(2.5), translate(-7.0)) == translate(-4.5)


def test_lens_examples():
    assert lens(50.0).apply(0.0, 0.2) == pytest.approx((0.0, 0.2))
    assert lens(50.0).apply(5.0, 0.0)[1] == pytest.approx(-0.1)
    assert lens(50.0, 5.0).apply(5.0, 0.0)[1] == pytest.approx(0.0)
    with pytest.raises(ValueError):
        lens(0.0)


def test_compose_invert_against_matrix_algebra():
    rng = np.random.default_rng(5)
    for _ in range(50):
        a = Affine1D(*rng.normal(size=6))
        b = Affine1D(*rng.normal(size=6))
        assert np.allclose(H(compose(a, b)), H(a) @ H(b), atol=1e-12)
        if abs(a.det()) > 1e-3:
            assert np.allclose(H(invert(a)), np.linalg.inv(H(a)), atol=1e-9)
    assert abs(lens(37.0, 1.5).det() - 1.0) < 1e-15
    assert abs(translate(13.0).det() - 1.0) < 1e-15


def test_in_focus_magnification_by_ray_tracing():
    """1/z + 1/D = 1/f: all rays from a scene point land at s = -(D/z) s0."""
    z, D = 300.0, 60.0
    X = compose(translate(D), compose(lens(F), translate(z)))
    for s0 in (-3.0, 0.0, 2.0):
        for u in (-0.02, 0.0, 0.013):
            assert X.apply(s0, u)[0] == pytest.approx(-(D / z) * s0, abs=1e-12)


def test_ray_coefficients_single_lens_closed_form():
    """lambda = -D/z (magnification), mu = 1 + D/z - D/f (0 iff thin-lens law)."""
    for z in (236.0, 280.0, 300.0, 364.0):
        D = 60.0
        q = Plane(16, 0.4, compose(lens(F), translate(z)))
        p = Plane(32, 0.04, translate(-D))
        lam, mu, nu = ray_coefficients(q, p)
        assert lam == pytest.approx(-D / z, rel=1e-13)
        assert mu == pytest.approx(1.0 + D / z - D / F, abs=1e-13)
        assert nu == 0.0
    lam, mu, nu = ray_coefficients(Plane(4, 1.0, compose(lens(F), translate(300.0))), Plane(4, 1.0, translate(-60.0)))
    assert abs(mu) < 1e-14


def test_degenerate_planes_rejected():
    with pytest.raises(DegenerateGeometry):  # source on the angular plane: b_q = 0
        ray_coefficients(Plane(4, 1.0, lens(F)), Plane(4, 1.0, translate(-60.0)))
    with pytest.raises(DegenerateGeometry):  # destination is the angular plane itself: lambda = 0
        ray_coefficients(Plane(4, 1.0, translate(-60.0)), Plane(4, 1.0, translate(0.0)))


# ----------------------------------------------------------- entries vs the exact inner product
def _geometries():
    """(src, dst) plane pairs of the kinds the cameras use."""
    out = []
    for z in (236.0, 280.0, 299.0, 300.5, 364.0):
        q = Plane(24, 0.4, compose(lens(F), translate(z)))
        out.append((q, Plane(48, 0.04, translate(-60.0))))          # slice -> single-lens detector
        out.append((q, Plane(40, 0.02, translate(-62.0))))          # slice -> lenslet array
    b, fmu, cmu = 0.413, 0.343, 0.16
    X0mu = compose(translate(-62.0), compose(invert(lens(fmu, cmu)), translate(-b)))
    out.append((Plane(40, 0.02, translate(-62.0)), Plane(64, 0.005, X0mu)))  # array -> detector via lenslet
    out.append((Plane(64, 0.005, X0mu), Plane(40, 0.02, translate(-62.0))))  # and back (adjoint direction)
    return out


def _inner_product_area(src, dst, i, j, s_k, d0):
    """<< b(dst cell i) a(angular cell k), b(src cell j) >> over (s,u) at the source plane."""
    Xpq = np.linalg.inv(H(dst.X0)) @ H(src.X0)
    P, Q, opq = Xpq[0]
    aq, bq, oq = src.X0.m00, src.X0.m01, src.X0.o0
    sj = src.centres()[j]
    si = dst.centres()[i]
    uc = (s_k - oq - aq * sj) / bq          # local origin to keep the coordinates small
    U = (d0 + abs(aq) * src.delta) / abs(bq) + 1e-9
    strips = [(aq, bq, s_k - oq - (aq * sj + bq * uc), d0),
              (P, Q, si - opq - (P * sj + Q * uc), dst.delta)]
    return strip_polygon_area(strips, (-0.5 * src.delta, 0.5 * src.delta, -U, U))


@pytest.mark.parametrize("g", range(len(_geometries())))
def test_pillbox_entries_match_polygon_area(g):
    src, dst = _geometries()[g]
    rng = np.random.default_rng(100 + g)
    d0 = 1.5
    worst = 0.0
    for s_k in (-5.25, -0.75, 2.25):
        lo, hi = band(src, dst, s_k, d0, PILLBOX)
        rows = [i for i in range(dst.n) if hi[i] >= lo[i]]
        for i in rng.choice(rows, size=min(12, len(rows)), replace=False):
            for j in range(max(lo[i] - 1, 0), min(hi[i] + 2, src.n)):
                ref = _inner_product_area(src, dst, i, j, s_k, d0)
                val = entries(src, dst, s_k, d0, PILLBOX, np.array([i]), np.array([j]))[0]
                scale = max(ref, 1e-300)
                if ref > 1e-12 * dst.delta * d0:
                    worst = max(worst, abs(val - ref) / scale)
                else:
                    assert abs(val) <= 1e-9 * dst.delta * d0 / abs(src.X0.m01)
    assert worst < 1e-9


def test_dirac_entries_match_interval_overlap():
    """Dirac angular basis: Delta0/|b_q| * |{s in cell j : |lam s + mu s_k + nu - s_i| <= Dp/2}|."""
    for src, dst in _geometries():
        lam, mu, nu = ray_coefficients(src, dst)
        d0 = 1.5
        for s_k in (-0.75, 2.25):
            M = transport_dense(src, dst, s_k, d0, DIRAC)
            sj, si = src.centres(), dst.centres()
            for i in range(0, dst.n, 7):
                a = (si[i] - 0.5 * dst.delta - mu * s_k - nu) / lam
                b = (si[i] + 0.5 * dst.delta - mu * s_k - nu) / lam
                a, b = min(a, b), max(a, b)
                for j in range(src.n):
                    ref = d0 / abs(src.X0.m01) * interval_overlap(a, b, sj[j] - 0.5 * src.delta, sj[j] + 0.5 * src.delta)
                    assert M[i, j] == pytest.approx(ref, rel=1e-9, abs=1e-15)


def test_symmetry_pq_qp():
    """B^{pq} = (B^{qp})^T, each side from its own closed form."""
    for src, dst in _geometries():
        for basis in (PILLBOX, DIRAC):
            for s_k in (-4.5, 0.0, 1.5):
                Bpq = transport_dense(src, dst, s_k, 1.5, basis)
                Bqp = transport_dense(dst, src, s_k, 1.5, basis)
                scale = np.abs(Bpq).max()
                assert np.abs(Bpq - Bqp.T).max() <= 1e-10 * scale


def test_identity_transport():
    """p = q with the same grid: B/V^p = I exactly (both bases)."""
    for X0 in (compose(lens(F), translate(280.0)), translate(-62.0)):
        p = Plane(20, 0.05, X0)
        for basis in (PILLBOX, DIRAC):
            B = transport_dense(p, p, 0.75, 1.5, basis) / basis_volume(p, 1.5)
            assert np.abs(B - np.eye(20)).max() < 1e-13


def test_basis_volume_by_polygon_area():
    """V^p = ||a b||^2 = area {|s| <= Dp/2} x {|X0p_s(s,u) - s_k| <= D0/2}."""
    for src, dst in _geometries():
        for p in (src, dst):
            a, b = p.X0.m00, p.X0.m01
            U = (1.5 + abs(a) * p.delta) / abs(b) + 1.0
            area = strip_polygon_area([(a, b, 0.0, 1.5)], (-0.5 * p.delta, 0.5 * p.delta, -U, U))
            assert basis_volume(p, 1.5) == pytest.approx(area, rel=1e-12)


def test_row_mass_equals_parallelogram_area():
    """sum_j B_ij over a full row = |{angular strip} cap {dest strip}| = D0 Dp / |det|."""
    for src, dst in _geometries():
        Xpq = np.linalg.inv(H(dst.X0)) @ H(src.X0)
        det = abs(src.X0.m00 * Xpq[0, 1] - src.X0.m01 * Xpq[0, 0])
        big = Plane(4000, src.delta, src.X0)    # wide source grid: every row is interior
        M = transport_sparse(big, dst, 0.75, 1.5, PILLBOX)
        mass = np.asarray(M.sum(axis=1)).ravel()
        assert np.allclose(mass, 1.5 * dst.delta / det, rtol=1e-12)


def test_angular_tiling_sums_to_full_aperture():
    """Sum over K pillbox cells tiling the aperture = one cell of the full width (tensor grid, Z4)."""
    for src, dst in _geometries():
        K, d0 = 8, 1.5
        centres = (np.arange(K) - (K - 1) * 0.5) * d0
        tot = sum(transport_dense(src, dst, sk, d0, PILLBOX) for sk in centres)
        full = transport_dense(src, dst, 0.0, K * d0, PILLBOX)
        assert np.abs(tot - full).max() <= 1e-12 * np.abs(full).max()


def test_in_focus_pillbox_is_dirac_rect():
    """mu = 0 (thin-lens law): the trapezoid collapses to the Dirac rect of height D0."""
    q = Plane(24, 0.4, compose(lens(F), translate(300.0)))
    p = Plane(48, 0.04, translate(-60.0))
    assert np.allclose(transport_dense(q, p, 1.0, 1.5, PILLBOX), transport_dense(q, p, 1.0, 1.5, DIRAC),
                       rtol=1e-10, atol=1e-15)


def test_band_contains_exactly_the_support():
    """The analytic band holds every nonzero entry and nothing outside it is nonzero (Z21)."""
    for src, dst in _geometries():
        M = transport_dense(src, dst, 0.75, 1.5, PILLBOX)
        lo, hi = band(src, dst, 0.75, 1.5, PILLBOX)
        for i in range(dst.n):
            nz = np.nonzero(M[i] > 1e-14 * np.abs(M).max())[0]
            if len(nz):
                assert lo[i] <= nz[0] and nz[-1] <= hi[i]
                assert hi[i] - lo[i] <= nz[-1] - nz[0] + 2


def test_separable_two_pass_equals_direct():
    """(B_s (x) B_t) via t-pass then s-pass == direct O(ST) sum over the 2D kernel."""
    rng = np.random.default_rng(3)
    src, dst = _geometries()[1]
    Bs = transport_dense(src, dst, 0.75, 1.5, PILLBOX)
    Bt = transport_dense(src, dst, -2.25, 1.5, PILLBOX)
    X = rng.random((src.n, src.n))                      # [t, s]
    two_pass = Bt @ X @ Bs.T
    direct = np.einsum("ik,jl,kl->ij", Bt, Bs, X)
    kron = (np.kron(Bt, Bs) @ X.ravel()).reshape(dst.n, dst.n)
    assert np.allclose(two_pass, direct, rtol=1e-13)
    assert np.allclose(two_pass, kron, rtol=1e-13)


def test_sparse_equals_dense():
    for src, dst in _geometries():
        for basis in (PILLBOX, DIRAC):
            D = transport_dense(src, dst, -1.5, 1.5, basis)
            S = transport_sparse(src, dst, -1.5, 1.5, basis).toarray()
            assert np.array_equal(D, S)


def test_row_params_trapezoid_widths():
    """Pillbox support half-width W and plateau w from the parallelogram geometry."""
    q = Plane(24, 0.4, compose(lens(F), translate(280.0)))
    p = Plane(48, 0.04, translate(-60.0))
    lam, mu, _ = ray_coefficients(q, p)
    c, W, w, Hh = row_params(q, p, 0.0, 1.5, PILLBOX)
    # the trapezoid is the overlap length of the angular cell with the dest-cell preimage (in s_0)
    xs = np.linspace(-1.2 * W, 1.2 * W, 201)
    ov = [interval_overlap(-0.75, 0.75, (-0.02 - lam * x) / mu, (0.02 - lam * x) / mu) if mu > 0 else
          interval_overlap(-0.75, 0.75, (0.02 - lam * x) / mu, (-0.02 - lam * x) / mu) for x in xs]
    from oracle.transport import trap_value
    assert np.allclose(trap_value(xs, W, w, Hh), ov, atol=1e-12)
    assert math.isclose(W, (1.5 * abs(mu) + 0.04) / (2 * abs(lam)), rel_tol=1e-14)
