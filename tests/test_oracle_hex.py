"""Pins for the oracle's non-separable lenslet stage (NEXT-4: hexagonal lenslet layout P:451, circular lenslet
apertures rasterised onto the array grid P:915-927; readings R12/R13).  CPU only.

* with a separable geometry the literal per-lenslet 2-D evaluation equals the separable per-axis form (the special
  case that reduces to the pinned model);
* dense A == matrix-free, fp64 adjoint identity;
* mask geometry: every array cell has at most one owner, odd rows sit half a pitch along s, and the open area of a
  finely rasterised disk converges to pi r^2;
* a point source through the hexagonal, circular-aperture camera matches an independent brute-force ray trace
  (lenslet found by testing the aperture disks themselves, not the oracle's masks).
"""
import math

import numpy as np
import pytest

from oracle.camera import CameraModel
from oracle.system import build_system
from workloads import make_config, normal_vector, uniform_volume
from workloads.geometry import plenoptic_camera


def test_2d_path_equals_separable_path():
    cam = plenoptic_camera(4, 8, 0.04, 2, 2, fill=0.75)
    sep = CameraModel(cam, (16, 16, 16), (0.4, 0.4, 0.4))
    two = CameraModel(dict(cam, _force_2d=True), (16, 16, 16), (0.4, 0.4, 0.4))
    assert two.nonsep and not sep.nonsep
    x = uniform_volume(dict(nx=16, ny=16, nz=16, dx=0.4, dy=0.4, dz=0.4), 0).astype(np.float64)
    y1, y2 = sep.forward(x), two.forward(x)
    assert np.abs(y1 - y2).max() <= 1e-12 * np.abs(y1).max()
    r = normal_vector(sep.n_pix, 3)
    g1, g2 = sep.adjoint(r), two.adjoint(r)
    assert np.abs(g1 - g2).max() <= 1e-12 * np.abs(g1).max()


@pytest.mark.parametrize("name", ["tiny_hex", "tiny_disk"])
def test_dense_and_adjoint(name):
    cfg = make_config(name)
    op = build_system(cfg)[0]
    A = op.dense()
    x = uniform_volume(cfg["volume"], 0).astype(np.float64).ravel()
    r = normal_vector(op.n_pix, 2).astype(np.float64)
    assert np.abs(A @ x - op.forward(x)).max() <= 1e-12 * np.abs(A @ x).max()
    assert np.abs(A.T @ r - op.adjoint(r)).max() <= 1e-12 * np.abs(A.T @ r).max()
    for seed in range(3):
        xx, rr = normal_vector(op.n_vox, 10 + seed), normal_vector(op.n_pix, 20 + seed)
        Ax = op.forward(xx)
        assert abs(Ax @ rr - xx @ op.adjoint(rr)) / (np.linalg.norm(Ax) * np.linalg.norm(rr)) <= 1e-10


def test_mask_geometry():
    cfg = make_config("tiny_hex")
    cam = build_system(cfg)[0].camera
    c = cfg["cameras"][0]
    ps, pt = c["n_s"] * c["px_s"] / c["nl_s"], c["n_t"] * c["px_t"] / c["nl_t"]
    owners = sum(m for *_, m in cam.lenslets2d)
    assert owners.max() == 1.0
    rows = {}
    for cs, ct, _, _, _ in cam.lenslets2d:
        rows.setdefault(round(ct / pt, 6), []).append(cs / ps)
    for k, (ct, cs) in enumerate(sorted(rows.items())):
        frac = [v - math.floor(v) for v in cs]
        want = 0.5 if k % 2 == 0 else 0.0          # nl_s = 4 (even): even rows at half-integers, odd rows shifted
        assert np.allclose(frac, want) and len(cs) == c["nl_s"] - (k % 2)
    # a finely rasterised disk of diameter fill * pitch_s: open area -> pi r^2 (cell-centre rule)
    fine = plenoptic_camera(4, 8, 0.04, 2, 32, lens_aperture=1, fill=0.8)
    m = CameraModel(fine, (16, 16, 16), (0.4, 0.4, 0.4)).lenslets2d[5][4]
    cell = (fine["n_s"] * fine["px_s"] / fine["nl_s"] / 32) ** 2
    area = m.sum() * cell
    r = 0.4 * fine["n_s"] * fine["px_s"] / fine["nl_s"]
    assert area == pytest.approx(math.pi * r * r, rel=0.03)


def _ray_trace_2d(cam, n_vox, vox, ix, iy, iz, n_rays=300000, seed=0):
    """Independent geometric ray trace through a lenslet array of any layout with circular apertures."""
    rng = np.random.default_rng(seed)
    z0 = cam["d_scene"] + (iz - (n_vox - 1) / 2) * vox
    p = np.stack([(ix - (n_vox - 1) / 2) * vox + (rng.random(n_rays) - 0.5) * vox,
                  (iy - (n_vox - 1) / 2) * vox + (rng.random(n_rays) - 0.5) * vox])
    z = z0 + (rng.random(n_rays) - 0.5) * vox
    p0 = np.stack([(rng.random(n_rays) - 0.5) * cam["ap_s"], (rng.random(n_rays) - 0.5) * cam["ap_t"]])
    f, D, b, fm = cam["f_main"], cam["d_mu_m"], cam["d_d_mu"], cam["f_mu"]
    u = (p0 - p) / z - p0 / f                       # slopes after the main lens
    pa = p0 + D * u                                 # hit points on the lenslet array
    ps, pt = cam["n_s"] * cam["px_s"] / cam["nl_s"], cam["n_t"] * cam["px_t"] / cam["nl_t"]
    centres = []
    for j in range(cam["nl_t"]):
        odd = cam["lens_layout"] == 1 and j % 2 == 1
        for i in range(cam["nl_s"] - (1 if odd else 0)):
            centres.append(((i - (cam["nl_s"] - 1) / 2 + (0.5 if odd else 0)) * ps, (j - (cam["nl_t"] - 1) / 2) * pt))
    centres = np.array(centres)
    r = 0.5 * cam["fill"] * ps
    d2 = (pa[0][:, None] - centres[None, :, 0]) ** 2 + (pa[1][:, None] - centres[None, :, 1]) ** 2
    mu = d2.argmin(1)
    if cam["aperture"] == 1:
        ok = d2[np.arange(n_rays), mu] < r * r
    else:
        ok = (np.abs(pa[0] - centres[mu, 0]) < 0.5 * cam["fill"] * ps) & (np.abs(pa[1] - centres[mu, 1]) < 0.5 * cam["fill"] * pt)
    c = centres[mu].T
    pd = pa + b * (u - (pa - c) / fm)               # lenslet, then propagate to the detector
    i_s = np.floor(pd[0] / cam["px_s"] + cam["n_s"] / 2.0).astype(int)
    i_t = np.floor(pd[1] / cam["px_t"] + cam["n_t"] / 2.0).astype(int)
    ok &= (i_s >= 0) & (i_s < cam["n_s"]) & (i_t >= 0) & (i_t < cam["n_t"])
    out = np.zeros((cam["n_t"], cam["n_s"]))
    np.add.at(out, (i_t[ok], i_s[ok]), 1.0)
    return out


def test_hex_point_source_matches_ray_trace():
    cam = plenoptic_camera(8, 16, 0.02, 8, 8, layout=1, lens_aperture=1, rows=9, px_per_row=14)
    n, vox = 16, 0.4
    model = CameraModel(cam, (n, n, n), (vox, vox, vox))
    for (ix, iy, iz) in ((9, 6, 4), (5, 8, 12)):
        x = np.zeros((n, n, n))
        x[iz, iy, ix] = 1.0
        ym = model.forward(x)
        rt = _ray_trace_2d(cam, n, vox, ix, iy, iz)
        ym, rt = ym / ym.sum(), rt / rt.sum()
        assert np.corrcoef(ym.ravel(), rt.ravel())[0, 1] > 0.85
        # energy in 8x8-pixel blocks and the image centroid
        eb_m = ym.reshape(cam["n_t"] // 14, 14, cam["n_s"] // 16, 16).sum((1, 3))
        eb_r = rt.reshape(cam["n_t"] // 14, 14, cam["n_s"] // 16, 16).sum((1, 3))
        assert np.abs(eb_m - eb_r).sum() < 0.12          # the cell-centre rasterisation of the disks costs ~0.08
        it, i_s = np.arange(cam["n_t"]), np.arange(cam["n_s"])
        assert (ym.sum(1) @ it) == pytest.approx(rt.sum(1) @ it, abs=1.0)
        assert (ym.sum(0) @ i_s) == pytest.approx(rt.sum(0) @ i_s, abs=1.0)


def test_circular_aperture_throughput_matches_ray_trace():
    """Energy through circular vs square lenslet apertures (fill 0.8, hexagonal rows, row pitch 0.875 of the column
    pitch): the model's ratio of total detector signal equals the ray trace's ratio of transmitted rays (exact disk
    and rectangle areas: ratio pi 0.4^2 / (0.8 x 0.7) = 0.898)."""
    n, vox = 16, 0.4
    ratios = []
    for kind in ("model", "rays"):
        tot = []
        for ap in (1, 0):
            # a fine array grid (n_a = 32 cells per lenslet) so the cell-centre rasterisation resolves the disk
            cam = plenoptic_camera(8, 16, 0.02, 4, 32, layout=1, lens_aperture=ap, rows=9, px_per_row=14, fill=0.8)
            if kind == "model":
                x = np.zeros((n, n, n))
                x[4:12, 4:12, 4:12] = 1.0
                tot.append(CameraModel(cam, (n, n, n), (vox, vox, vox)).forward(x).sum())
            else:
                tot.append(sum(_ray_trace_2d(cam, n, vox, ix, iy, iz, n_rays=60000, seed=ix + 16 * iy + 256 * iz).sum()
                               for ix in (5, 8, 11) for iy in (5, 8, 11) for iz in (5, 8, 11)))
        ratios.append(tot[0] / tot[1])
    assert ratios[0] == pytest.approx(ratios[1], rel=0.04)
    assert 0.85 < ratios[0] < 0.95
