"""Pins for oracle/camera.py and oracle/system.py (CPU only).

* explicit dense A (Kronecker assembly) == matrix-free factored evaluation;
* fp64 adjoint dot test <Ax,y> = <x,A^T y> to 1e-10 (north star);
* factored plenoptic chain == unfactored per-lenslet, per-slice sum;
* single-lens in-focus point source: image centroid at the magnified position
  -(D/z) x0;
* plenoptic: the model image of a point source matches an independent brute-force
  ray trace (main lens -> lenslet array -> detector) sub-image by sub-image;
* mask: fill 0 blocks everything.
"""
import math

import numpy as np
import pytest

from oracle.camera import CameraModel
from oracle.system import SystemOperator, build_system
from workloads import make_config, normal_vector, uniform_volume
from workloads.geometry import plenoptic_camera, single_camera

TINY = ["tiny", "tiny_k4", "tiny_single", "tiny_yaw15", "tiny_dirac", "tiny_turn"]


@pytest.mark.parametrize("name", TINY)
def test_dense_equals_matrix_free(name):
    cfg = make_config(name)
    op = build_system(cfg)[0]
    A = op.dense()
    x = uniform_volume(cfg["volume"], 0).astype(np.float64).ravel()
    r = normal_vector(op.n_pix, 2).astype(np.float64)
    y = op.forward(x)
    assert np.abs(A @ x - y).max() <= 1e-12 * np.abs(y).max()
    g = op.adjoint(r)
    assert np.abs(A.T @ r - g).max() <= 1e-12 * np.abs(g).max()


@pytest.mark.parametrize("name", TINY + ["small_two"])
def test_adjoint_dot_fp64(name):
    cfg = make_config(name)
    for op in build_system(cfg):
        for seed in range(3):
            x = normal_vector(op.n_vox, 10 + seed).astype(np.float64)
            r = normal_vector(op.n_pix, 20 + seed).astype(np.float64)
            Ax = op.forward(x)
            err = abs(Ax @ r - x @ op.adjoint(r)) / (np.linalg.norm(Ax) * np.linalg.norm(r))
            assert err <= 1e-10


def test_factored_equals_unfactored():
    cfg = make_config("tiny")
    vol = cfg["volume"]
    cam = CameraModel(cfg["cameras"][0], (16, 16, 16), (vol["dx"], vol["dy"], vol["dz"]))
    x = uniform_volume(vol, 0).astype(np.float64)
    y_f = cam.forward(x)
    from oracle.transport import transport_sparse
    y_u = np.zeros_like(y_f)
    for ks in range(cam.ks):
        for kt in range(cam.kt):
            for n in range(cam.nz):
                a_n = cam.scale_s1 * (cam.S1[1][kt][n] @ x[n] @ cam.S1[0][ks][n].T)
                for mus, pls in enumerate(cam.lenslet_planes[0]):
                    Bs = transport_sparse(cam.array_planes[0], pls, cam.sk[0][ks], cam.d0[0], cam.basis)
                    Bs = Bs.toarray() * cam.masks[0][mus][None, :]
                    for mut, plt in enumerate(cam.lenslet_planes[1]):
                        Bt = transport_sparse(cam.array_planes[1], plt, cam.sk[1][kt], cam.d0[1], cam.basis)
                        Bt = Bt.toarray() * cam.masks[1][mut][None, :]
                        y_u += cam.scale_s3 * (Bt @ a_n @ Bs.T)
    assert np.abs(y_f - y_u).max() <= 1e-12 * np.abs(y_f).max()


def test_blocking_mask_gives_zero():
    cam = plenoptic_camera(4, 8, 0.04, 2, 2, fill=0.0)
    model = CameraModel(cam, (16, 16, 16), (0.4, 0.4, 0.4))
    assert np.all(model.forward(np.ones((16, 16, 16))) == 0.0)


def test_single_lens_in_focus_centroid():
    cam = single_camera(64, 0.04, 4)
    model = CameraModel(cam, (16, 16, 16), (0.4, 0.4, 0.4))
    xs = (np.arange(16) - 7.5) * 0.4
    det = (np.arange(64) - 31.5) * 0.04
    for ix, iy in ((3, 12), (10, 5)):
        x = np.zeros((16, 16, 16))
        x[8, iy, ix] = 1.0            # slice 8 is at z = 300.2, ~in focus (D = 60)
        y = model.forward(x)
        z = model.z[8]
        cs = (y.sum(0) * det).sum() / y.sum()
        ct = (y.sum(1) * det).sum() / y.sum()
        assert cs == pytest.approx(-(60.0 / z) * xs[ix], abs=0.04)
        assert ct == pytest.approx(-(60.0 / z) * xs[iy], abs=0.04)


def _ray_trace(cam, n_vox, vox, ix, iy, iz, n_rays=400000, seed=0):
    """Independent geometric ray trace of one voxel through a plenoptic camera (test-side)."""
    rng = np.random.default_rng(seed)
    z0 = cam["d_scene"] + (iz - (n_vox - 1) / 2) * vox
    xs0 = (ix - (n_vox - 1) / 2) * vox
    ys0 = (iy - (n_vox - 1) / 2) * vox
    s = xs0 + (rng.random(n_rays) - 0.5) * vox
    t = ys0 + (rng.random(n_rays) - 0.5) * vox
    z = z0 + (rng.random(n_rays) - 0.5) * vox
    s0 = (rng.random(n_rays) - 0.5) * cam["ap_s"]     # aperture position (angular plane)
    t0 = (rng.random(n_rays) - 0.5) * cam["ap_t"]
    f, D, b, fm = cam["f_main"], cam["d_mu_m"], cam["d_d_mu"], cam["f_mu"]
    pitch = cam["n_s"] * cam["px_s"] / cam["nl_s"]
    out = np.zeros((cam["n_t"], cam["n_s"]))
    for pos0, pos, axis in ((s0, s, 0), (t0, t, 1)):
        u = (pos0 - pos) / z                   # slope from the scene point to the aperture point
        u = u - pos0 / f                        # main lens
        pa = pos0 + D * u                       # at the array
        mu = np.floor(pa / pitch + cam["nl_s"] / 2.0)
        c = (mu - (cam["nl_s"] - 1) / 2.0) * pitch
        ok = (mu >= 0) & (mu < cam["nl_s"])
        u2 = u - (pa - c) / fm                 # lenslet
        pd = pa + b * u2
        if axis == 0:
            ps, oks = pd, ok
        else:
            pt, okt = pd, ok
    ok = oks & okt
    i_s = np.floor(ps / cam["px_s"] + cam["n_s"] / 2.0).astype(int)
    i_t = np.floor(pt / cam["px_t"] + cam["n_t"] / 2.0).astype(int)
    ok &= (i_s >= 0) & (i_s < cam["n_s"]) & (i_t >= 0) & (i_t < cam["n_t"])
    np.add.at(out, (i_t[ok], i_s[ok]), 1.0)
    return out


def test_plenoptic_point_source_matches_ray_trace():
    """Sub-image centroids and per-lenslet energy of the model vs a brute-force ray trace."""
    cam = plenoptic_camera(8, 16, 0.02, 8, 8)
    n, vox = 16, 0.4
    model = CameraModel(cam, (n, n, n), (vox, vox, vox))
    for (ix, iy, iz) in ((9, 6, 4), (5, 8, 12)):
        x = np.zeros((n, n, n))
        x[iz, iy, ix] = 1.0
        y = model.forward(x)
        rt = _ray_trace(cam, n, vox, ix, iy, iz)
        ym = y / y.sum()
        rtm = rt / rt.sum()
        L = 16
        e_m = ym.reshape(8, L, 8, L).sum((1, 3))
        e_r = rtm.reshape(8, L, 8, L).sum((1, 3))
        assert np.abs(e_m - e_r).sum() < 0.03        # energy per lenslet sub-image
        assert np.corrcoef(ym.ravel(), rtm.ravel())[0, 1] > 0.85
        coords = np.arange(L)
        for a in range(8):
            for b in range(8):
                if e_r[a, b] > 0.05:
                    sm, sr = ym[a*L:(a+1)*L, b*L:(b+1)*L], rtm[a*L:(a+1)*L, b*L:(b+1)*L]
                    assert (sm.sum(0) @ coords) / sm.sum() == pytest.approx((sr.sum(0) @ coords) / sr.sum(), abs=1.0)
                    assert (sm.sum(1) @ coords) / sm.sum() == pytest.approx((sr.sum(1) @ coords) / sr.sum(), abs=1.0)
