"""Pins for oracle/rotation.py (CPU only): factor re-multiplication, the yaw closed form,
the shear entries by brute-force quadrature of the L2-projection overlap integral
(P:1165-1171), row sums / transpose / identity invariants, and rotation fidelity of a
smooth blob against the analytic rotation f(Theta p^r)."""
import json
import math
import os

import numpy as np
import pytest

from oracle.rotation import NotDecomposable, Rotation, decompose, factor_matrices, shear_kernel, shear_matrix
from tests.brute import quad2
from workloads.geometry import pose_pitch, pose_yaw, pose_yaw_pitch

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def _random_rotation(rng, max_deg):
    axis = rng.normal(size=3)
    axis /= np.linalg.norm(axis)
    ang = math.radians(rng.uniform(-max_deg, max_deg))
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * K @ K


def test_factors_reproduce_theta():
    rng = np.random.default_rng(11)
    for _ in range(500):
        R = _random_rotation(rng, 30.0)
        D, Sz, Sx, Sy = factor_matrices(decompose(R.ravel()))
        assert np.abs(D @ Sz @ Sx @ Sy - R).max() < 1e-14


def test_yaw_and_pitch_golden():
    for key, pose in (("yaw30", pose_yaw(30.0)), ("pitch30", pose_pitch(30.0))):
        ref = GOLDEN["rotation"][key]
        dec = decompose(pose)
        assert np.allclose(dec["D"], ref["D"], atol=1e-6)
        for k, v in ref["shears"].items():
            assert dec[k] == pytest.approx(v, abs=1e-6)


def test_yaw_closed_form():
    for deg in (5.0, 15.0, 30.0, 44.0):
        th = math.radians(deg)
        dec = decompose(pose_yaw(deg))
        assert np.allclose(dec["D"], (math.cos(th), 1.0, 1.0 / math.cos(th)), rtol=1e-14)
        assert dec["a_zx"] == pytest.approx(-math.sin(th) * math.cos(th), abs=1e-15)
        assert dec["a_xz"] == pytest.approx(math.tan(th), rel=1e-14)
        for k in ("a_yx", "a_yz", "a_xy", "a_zy"):
            assert dec[k] == 0.0


def test_quarter_turn_rejected():
    with pytest.raises(NotDecomposable):
        decompose(pose_yaw(90.0))


def test_quarter_turn_choice():
    """Reading R7: P is a proper cube rotation, P Theta' reproduces Theta, and the residual angle is the
    smallest over the 24 candidates (<= 45 deg for single-axis poses; identity below 45 deg)."""
    from oracle.rotation import _proper_signed_permutations, quarter_turn
    assert len(_proper_signed_permutations()) == 24
    for pose, resid in ((pose_yaw(30.0), 30.0), (pose_yaw(50.0), 40.0), (pose_yaw(120.0), 30.0),
                        (pose_pitch(100.0), 10.0), (pose_yaw(-135.0), 45.0), (pose_yaw(90.0), 0.0)):
        P, T = quarter_turn(pose)
        assert abs(np.linalg.det(P) - 1.0) < 1e-15 and set(np.abs(P).ravel()) <= {0.0, 1.0}
        assert np.abs(P @ T - np.asarray(pose).reshape(3, 3)).max() < 1e-15
        ang = np.degrees(np.arccos(np.clip((np.trace(T) - 1) / 2, -1, 1)))
        assert ang == pytest.approx(resid, abs=1e-9)
    assert np.array_equal(quarter_turn(pose_yaw(30.0))[0], np.eye(3))


def test_quarter_turn_is_exact_relabelling():
    """A 90-degree yaw is a pure permutation of the voxels: x^r equals the point samples of the rotated
    blob exactly (p = Theta p^r), and the adjoint is its transpose."""
    n, d = 12, 0.4
    c = (np.arange(n) - (n - 1) / 2) * d
    x = _gauss_cell_average((c, c, c))
    for pose in (pose_yaw(90.0), pose_yaw(-90.0), pose_pitch(90.0), pose_yaw(180.0)):
        rot = Rotation(pose, (n, n, n), (d, d, d))
        ref = _gauss_cell_average((c, c, c), R=pose)
        assert np.abs(rot.forward(x) - ref).max() < 1e-12
        rng = np.random.default_rng(1)
        a, b = rng.normal(size=(n, n, n)), rng.normal(size=(n, n, n))
        assert abs(np.sum(rot.forward(a) * b) - np.sum(a * rot.adjoint(b))) < 1e-12 * np.linalg.norm(a) * np.linalg.norm(b)


def test_quarter_turn_needs_equal_axes():
    with pytest.raises(NotDecomposable):
        Rotation(pose_yaw(90.0), (8, 8, 10), (0.4, 0.4, 0.4))


@pytest.mark.parametrize("wa,wb", [(0.0, 0.0), (0.35, 0.0), (0.0, 0.8), (0.3, 0.55), (0.9, 0.9), (1.7, 0.2)])
def test_shear_kernel_vs_quadrature(wa, wb):
    """E entry = 1/(Dx Dy Dz) int int Lambda_Dz(d - a xi - b eta) over the cell (brute force)."""
    Dz = 0.35
    lam = lambda t: np.maximum(0.0, Dz - np.abs(t))
    for d in np.linspace(-1.2, 1.2, 17):
        if wa == 0.0 and wb == 0.0:
            ref = lam(d) / Dz
        else:
            ref = quad2(lambda xi, eta: lam(d - wa * xi - wb * eta), -0.5, 0.5, -0.5, 0.5, n=800) / Dz
        assert shear_kernel(d, Dz, wa, wb) == pytest.approx(ref, abs=2e-6)


def _pose_dec(pose):
    return decompose(pose)


def test_shear_invariants():
    dims, vox = (9, 8, 10), (0.46, 0.4, 0.35)
    for axis, c in (("z", (-0.43, 0.2)), ("x", (0.1, 0.57)), ("y", (0.3, -0.2))):
        E = shear_matrix(dims, vox, axis, *c).toarray()
        Em = shear_matrix(dims, vox, axis, -c[0], -c[1]).toarray()
        assert np.abs(E.T - Em).max() < 1e-13               # E(a,b)^T = E(-a,-b)
        assert np.abs(shear_matrix(dims, vox, axis, 0.0, 0.0).toarray() - np.eye(E.shape[0])).max() < 1e-15
        # interior rows sum to 1 (partition of unity of the voxel basis)
        big = shear_matrix((40, 40, 40), vox, axis, *c)
        rs = np.asarray(big.sum(axis=1)).ravel().reshape(40, 40, 40)
        assert np.abs(rs[15:25, 15:25, 15:25] - 1.0).max() < 1e-12
        assert (E >= -1e-16).all()


BLOB_C = np.array([1.2, -0.8, 0.6])
BLOB_S = np.array([1.0, 1.6, 2.4])


def _gauss_cell_average(centres, R=None):
    """Anisotropic off-centre blob f(p) at p = R p^r, point samples (smooth relative to the cells)."""
    Z, Y, X = np.meshgrid(*centres[::-1], indexing="ij")
    P = np.stack([X, Y, Z], -1)
    if R is not None:
        P = P @ np.asarray(R).reshape(3, 3).T
    return np.exp(-0.5 * np.sum(((P - BLOB_C) / BLOB_S) ** 2, -1))


@pytest.mark.parametrize("pose", [pose_yaw(20.0), pose_yaw(30.0), pose_pitch(25.0), pose_yaw_pitch(20.0, 15.0),
                                  pose_yaw(120.0), pose_pitch(-100.0), pose_yaw_pitch(70.0, 50.0)])
def test_rotation_fidelity_blob(pose):
    n, d = 40, 0.4
    c = (np.arange(n) - (n - 1) / 2) * d
    x = _gauss_cell_average((c, c, c))
    rot = Rotation(pose, (n, n, n), (d, d, d))
    xr = rot.forward(x)
    cr = [(np.arange(n) - (n - 1) / 2) * v for v in rot.vox_r]
    ref = _gauss_cell_average(cr, R=pose)
    nrmse = np.linalg.norm(xr - ref) / np.linalg.norm(ref)
    assert nrmse < 0.05
    # the wrong sense of rotation is clearly worse (pins the direction convention)
    wrong = _gauss_cell_average(cr, R=np.asarray(pose).reshape(3, 3).T.ravel())
    assert np.linalg.norm(xr - wrong) / np.linalg.norm(wrong) > 2 * nrmse


def test_rotation_adjoint_is_transpose():
    rot = Rotation(pose_yaw_pitch(25.0, -10.0), (7, 6, 8), (0.4, 0.4, 0.4))
    rng = np.random.default_rng(0)
    x, y = rng.normal(size=(8, 6, 7)), rng.normal(size=(8, 6, 7))
    lhs = np.sum(rot.forward(x) * y)
    rhs = np.sum(x * rot.adjoint(y))
    assert abs(lhs - rhs) < 1e-12 * np.linalg.norm(x) * np.linalg.norm(y)
