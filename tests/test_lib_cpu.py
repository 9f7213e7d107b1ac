"""CPU checks of the C-ABI library (no GPU needed): it loads, exports every symbol include/lfm.h
declares, and a host-only plan (cuda_device = -1) reproduces the oracle's index/geometry tables
bit-exactly (north star: "bit-exactly on index/geometry tables") and its fp64 weights.

The oracle computes its bands from its own closed form (oracle/transport.py); the plan computes
them independently in C++ (paper_1812_03358_b200/csrc/plan.cpp); both follow the op order of
DESIGN.md reading Z21."""
import ctypes
import re

import numpy as np
import pytest

from oracle.rotation import decompose, shear_matrix
from oracle.system import build_system
from oracle.transport import band, basis_volume
from workloads import make_config
from workloads.geometry import plenoptic_camera, pose_yaw, pose_yaw_pitch, single_camera

lfm = pytest.importorskip("paper_1812_03358_b200.lfm")

CONFIGS = ["tiny", "tiny_k4", "tiny_single", "tiny_yaw15", "tiny_multi", "tiny_dirac", "tiny_turn", "small_two"]


def ragged_config():
    cam = plenoptic_camera(5, 7, 0.05, 3, 2, pose=pose_yaw_pitch(12.0, -7.0))
    cam.update(nl_t=3, n_t=21, k_t=2)
    return dict(name="ragged", volume=dict(nx=19, ny=17, nz=13, dx=0.45, dy=0.4, dz=0.35),
                cameras=[cam, single_camera(23, 0.05, 3, pose=pose_yaw_pitch(-20.0, 10.0))])


def _cfg(name):
    return ragged_config() if name == "ragged" else make_config(name)


def test_exports_every_header_symbol():
    header = open(lfm.os.path.join(lfm._HERE, "..", "include", "lfm.h")).read()
    names = sorted(set(re.findall(r"^\s*(?:lfm_status|int|const char\*)\s+(lfm_\w+)\s*\(", header, re.M)))
    assert len(names) >= 16
    lib = ctypes.CDLL(lfm.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(lfm.EXPORTED)
    assert lfm.version().startswith("liblfm")


def test_binding_constants_match_header():
    """Every #define LFM_<NAME> <int> of include/lfm.h that the binding mirrors has the same value there."""
    header = open(lfm.os.path.join(lfm._HERE, "..", "include", "lfm.h")).read()
    defs = {k: int(v) for k, v in re.findall(r"^#define\s+LFM_(\w+)\s+(-?\d+)\s*$", header, re.M)}
    mirrored = {"MAJ_SUM": lfm.MAJ_SUM, "MAJ_FINISH": lfm.MAJ_FINISH, "GRAD_ACCUMULATE": lfm.GRAD_ACCUMULATE}
    for k, v in mirrored.items():
        assert defs[k] == v, k


def _oracle_s3_band(cam, ax, k):
    """Union over lenslets of band_mu(i) cap open cells of mu (reading Z9/Z10)."""
    n_det = cam.lenslet_planes[ax][0].n
    lo = np.full(n_det, 1 << 30)
    hi = np.full(n_det, -1)
    for mu, pl in enumerate(cam.lenslet_planes[ax]):
        open_cells = np.nonzero(cam.masks[ax][mu])[0]
        if len(open_cells) == 0:
            continue
        blo, bhi = band(cam.array_planes[ax], pl, cam.sk[ax][k], cam.d0[ax], cam.basis)
        blo = np.maximum(blo, open_cells[0])
        bhi = np.minimum(bhi, open_cells[-1])
        ok = bhi >= blo
        lo = np.where(ok, np.minimum(lo, blo), lo)
        hi = np.where(ok, np.maximum(hi, bhi), hi)
    empty = hi < 0
    return np.where(empty, 0, lo), np.where(empty, 0, hi - lo + 1)


def _bands_equal(plan, c, tab, ax, idx, lo, hi):
    st = plan.export_table(c, tab + "_START", ax, idx)
    ln = plan.export_table(c, tab + "_LEN", ax, idx)
    ln_o = np.where(hi >= lo, hi - lo + 1, 0)
    st_o = np.where(hi >= lo, lo, 0)
    assert np.array_equal(st, st_o) and np.array_equal(ln, ln_o), (tab, ax, idx)
    return st, ln


def _weights_match(plan, c, tab, ax, idx, dense, rel=1e-13):
    st = plan.export_table(c, tab + "_START", ax, idx)
    ln = plan.export_table(c, tab + "_LEN", ax, idx)
    w = plan.export_table(c, tab + "_W64", ax, idx).reshape(len(st), -1)
    rec = np.zeros_like(dense)
    for i in range(len(st)):
        rec[i, st[i]:st[i] + ln[i]] = w[i, :ln[i]]
    scale = max(np.abs(dense).max(), 1e-300)
    assert np.abs(rec - dense).max() <= rel * scale, (tab, ax, idx)


@pytest.mark.parametrize("name", CONFIGS + ["ragged"])
def test_band_tables_bit_exact(name):
    cfg = _cfg(name)
    plan = lfm.Plan(cfg, device=-1)
    for c, op in enumerate(build_system(cfg)):
        cam = op.camera
        dst = cam.array_planes if cam.type == 1 else cam.det_planes
        for ax in range(2):
            for k in range(len(cam.sk[ax])):
                for n in range(cam.nz):
                    idx = k * cam.nz + n
                    lo, hi = band(cam.slice_planes[ax][n], dst[ax], cam.sk[ax][k], cam.d0[ax], cam.basis)
                    _bands_equal(plan, c, "S1F", ax, idx, lo, hi)
                    _weights_match(plan, c, "S1F", ax, idx, cam.S1[ax][k][n].toarray())
                    lo, hi = band(dst[ax], cam.slice_planes[ax][n], cam.sk[ax][k], cam.d0[ax], cam.basis)
                    _bands_equal(plan, c, "S1A", ax, idx, lo, hi)
                    # adjoint table = the transport in the other direction = transpose
                    _weights_match(plan, c, "S1A", ax, idx, cam.S1[ax][k][n].toarray().T, rel=1e-10)
                if cam.type == 1:
                    st_o, ln_o = _oracle_s3_band(cam, ax, k)
                    assert np.array_equal(plan.export_table(c, "S3F_START", ax, k), st_o)
                    assert np.array_equal(plan.export_table(c, "S3F_LEN", ax, k), ln_o)
                    _weights_match(plan, c, "S3F", ax, k, cam.S3[ax][k].toarray())
                    _weights_match(plan, c, "S3A", ax, k, cam.S3[ax][k].toarray().T, rel=1e-10)


@pytest.mark.parametrize("name", ["tiny", "tiny_single", "tiny_dirac", "small_two", "ragged"])
def test_collapsed_composite_tables(name):
    """C_n = sum_k S_k B_{k,n} per axis (exact re-association over the tensor angular grid)."""
    cfg = _cfg(name)
    plan = lfm.Plan(cfg, device=-1)
    for c, op in enumerate(build_system(cfg)):
        cam = op.camera
        for ax in range(2):
            for n in range(cam.nz):
                Cn = 0
                for k in range(len(cam.sk[ax])):
                    B = cam.S1[ax][k][n]
                    Cn = Cn + ((cam.S3[ax][k] @ B) if cam.type == 1 else B)
                Cn = Cn.toarray()
                nz = Cn > 0
                lo = np.where(nz.any(1), nz.argmax(1), 0)
                hi = np.where(nz.any(1), Cn.shape[1] - 1 - nz[:, ::-1].argmax(1), -1)
                _bands_equal(plan, c, "CF", ax, n, lo, hi)
                _weights_match(plan, c, "CF", ax, n, Cn, rel=1e-12)


@pytest.mark.parametrize("name", ["tiny_yaw15", "ragged", "small_two", "tiny_turn"])
def test_rotation_factors_and_shear_tables(name):
    from oracle.rotation import quarter_turn
    cfg = _cfg(name)
    plan = lfm.Plan(cfg, device=-1)
    vol = cfg["volume"]
    dims = (vol["nx"], vol["ny"], vol["nz"])
    vox = (vol["dx"], vol["dy"], vol["dz"])
    for c, cam in enumerate(cfg["cameras"]):
        inf = plan.info(c)
        P, T = quarter_turn(cam["R"])                                 # reading R7
        assert inf["rot_perm"] == [int(v) for v in P.ravel()]
        assert bool(inf["rot_passes"] & 8) == (not np.array_equal(P, np.eye(3)))
        dec = decompose(T.ravel())
        assert tuple(inf["rot_D"]) == dec["D"]                       # bit-exact fp64 geometry
        assert tuple(inf["shear"]) == (dec["a_zx"], dec["a_zy"], dec["a_xy"], dec["a_xz"], dec["a_yx"], dec["a_yz"])
        vox_r = tuple(v / d for v, d in zip(vox, dec["D"]))
        assert tuple(inf["vox_r"]) == vox_r
        coeffs = [(dec["a_zx"], dec["a_zy"]), (dec["a_xy"], dec["a_xz"]), (dec["a_yx"], dec["a_yz"])]
        import scipy.sparse as sp
        for p, axis in enumerate("zxy"):
            E = shear_matrix(dims, vox_r, axis, *coeffs[p]).tocsr()
            mlo = plan.export_table(c, "ROT_MLO", 0, p)
            if len(mlo) == 0:                                        # identity pass skipped
                assert coeffs[p] == (0.0, 0.0)
                continue
            w = plan.export_table(c, "ROT_W64", 0, p).reshape(len(mlo), -1)
            nx, ny, nz = dims
            flat = np.arange(nx * ny * nz)
            ix, iy, iz = flat % nx, (flat // nx) % ny, flat // (nx * ny)
            line, pos, n, stride = {"z": (ix + nx * iy, iz, nz, nx * ny), "x": (iy + ny * iz, ix, nx, 1),
                                    "y": (ix + nx * iz, iy, ny, nx)}[axis]
            rows, cols, vals = [], [], []
            for q in range(w.shape[1]):                              # the plan's line tables as a sparse matrix
                j = pos + mlo[line] + q
                ok = (j >= 0) & (j < n) & (w[line, q] != 0.0)
                rows.append(flat[ok]); cols.append((flat + (j - pos) * stride)[ok]); vals.append(w[line, q][ok])
            N = nx * ny * nz
            rec = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))
            assert abs(rec - E).max() <= 1e-12


@pytest.mark.parametrize("name", CONFIGS)
def test_scalars_match_oracle(name):
    cfg = _cfg(name)
    plan = lfm.Plan(cfg, device=-1)
    for c, op in enumerate(build_system(cfg)):
        sc = plan.export_table(c, "SCALARS", 0, 0)
        cam = op.camera
        assert sc[0] == pytest.approx(cam.scale_s1, rel=1e-14)
        if cam.type == 1:
            assert sc[1] == pytest.approx(cam.scale_s3, rel=1e-14)
            assert sc[2] == pytest.approx(basis_volume(cam.array_planes[0], cam.d0[0]) *
                                          basis_volume(cam.array_planes[1], cam.d0[1]), rel=1e-14)


def test_error_statuses():
    vol = dict(nx=8, ny=8, nz=8, dx=0.4, dy=0.4, dz=0.4)
    cases = [
        (plenoptic_camera(4, 8, 0.04, 2, 2, fill=1.5), 1),           # fill > 1
        (dict(single_camera(32, 0.04, 2), f_main=0.0), 2),           # zero focal length
        (dict(single_camera(32, 0.04, 2), d_det=0.0), 3),            # detector on the angular plane
        (dict(single_camera(32, 0.04, 2), k_s=0), 1),
    ]
    for cam, status in cases:
        with pytest.raises(lfm.LfmError) as e:
            lfm.Plan(dict(volume=vol, cameras=[cam]), device=-1)
        assert e.value.status == status, (cam, e.value)
        assert "camera 0" in str(e.value)
    # a quarter turn is an exact relabelling only between equal axes (reading R7)
    vol2 = dict(nx=8, ny=8, nz=10, dx=0.4, dy=0.4, dz=0.4)
    with pytest.raises(lfm.LfmError) as e:
        lfm.Plan(dict(volume=vol2, cameras=[plenoptic_camera(4, 8, 0.04, 2, 2, pose=pose_yaw(90.0))]), device=-1)
    assert e.value.status == 3 and "quarter-turn" in str(e.value)
    lfm.Plan(dict(volume=vol, cameras=[plenoptic_camera(4, 8, 0.04, 2, 2, pose=pose_yaw(90.0))]), device=-1)
    with pytest.raises(lfm.LfmError) as e:
        lfm.Plan(dict(volume=vol, cameras=[]), device=-1)
    assert e.value.status == 1


def test_host_only_plan_rejects_apply_calls():
    plan = lfm.Plan(make_config("tiny"), device=-1)
    assert plan.info(0)["ws_bytes"] > 0
    import torch
    ws = torch.empty(plan.ws_bytes, dtype=torch.uint8)
    x = torch.zeros(plan.info(0)["n_vox"])
    y = torch.zeros(plan.info(0)["n_pix"])
    with pytest.raises(lfm.LfmError) as e:
        lfm.A_forward(plan, 0, x, y, ws, stream=0)
    assert e.value.status == 1 and "host-only" in str(e.value)


def test_tables_bit_exact_at_128():
    """The metric's config (128^3 two-camera, 2048^2 detectors, K = 8x8): every S1 band (both directions, both
    axes, all 8 views x 128 slices), every S3 band, the rotation factors of the 30-degree camera bit-exact;
    weights (fp64) on every 16th slice and the collapsed composite on 3 slices (bit-exact tables were
    checked only on tiny/small configs)."""
    from oracle.rotation import quarter_turn
    cfg = make_config("128^3 two-camera")
    plan = lfm.Plan(cfg, device=-1)
    for c, op in enumerate(build_system(cfg)):
        cam = op.camera
        inf = plan.info(c)
        P, T = quarter_turn(cfg["cameras"][c]["R"])
        dec = decompose(T.ravel())
        assert tuple(inf["rot_D"]) == dec["D"]
        assert tuple(inf["shear"]) == (dec["a_zx"], dec["a_zy"], dec["a_xy"], dec["a_xz"], dec["a_yx"], dec["a_yz"])
        dst = cam.array_planes
        for ax in range(2):
            for k in range(len(cam.sk[ax])):
                for n in range(cam.nz):
                    idx = k * cam.nz + n
                    lo, hi = band(cam.slice_planes[ax][n], dst[ax], cam.sk[ax][k], cam.d0[ax], cam.basis)
                    _bands_equal(plan, c, "S1F", ax, idx, lo, hi)
                    lo, hi = band(dst[ax], cam.slice_planes[ax][n], cam.sk[ax][k], cam.d0[ax], cam.basis)
                    _bands_equal(plan, c, "S1A", ax, idx, lo, hi)
                    if n % 16 == 5:
                        _weights_match(plan, c, "S1F", ax, idx, cam.S1[ax][k][n].toarray())
                st_o, ln_o = _oracle_s3_band(cam, ax, k)
                assert np.array_equal(plan.export_table(c, "S3F_START", ax, k), st_o)
                assert np.array_equal(plan.export_table(c, "S3F_LEN", ax, k), ln_o)
            _weights_match(plan, c, "S3F", ax, 3, cam.S3[ax][3].toarray())
            for n in (0, 64, 127):
                # composite band (reading Z21): the union of the S1 bands of every array cell that a non-zero S3
                # entry of the row reaches, over all views.  Both sides decide "non-zero" on their own fp64 S3
                # evaluation, and at a few trapezoid edges one side leaves rounding residue (1e-24..1e-30 of the
                # row's entries) where the other gives exactly 0.  So: the plan's band equals the oracle's on
                # every row where the residue does not matter, and elsewhere lies between the band of the
                # oracle's significant entries (> 1e-20 of max) and that of all its non-zero entries.
                Cn = 0
                n_det = cam.S3[ax][0].shape[0]
                lo = {m: np.full(n_det, 1 << 30) for m in ("sig", "any")}
                hi = {m: np.full(n_det, -1) for m in ("sig", "any")}
                for k in range(len(cam.sk[ax])):
                    Cn = Cn + cam.S3[ax][k] @ cam.S1[ax][k][n]
                    b_lo, b_hi = band(cam.slice_planes[ax][n], dst[ax], cam.sk[ax][k], cam.d0[ax], cam.basis)
                    s3 = cam.S3[ax][k].tocoo()
                    for m, keep in (("sig", np.abs(s3.data) > 1e-20 * np.abs(s3.data).max()), ("any", s3.data != 0.0)):
                        keep = keep & (b_hi[s3.col] >= b_lo[s3.col])
                        np.minimum.at(lo[m], s3.row[keep], b_lo[s3.col[keep]])
                        np.maximum.at(hi[m], s3.row[keep], b_hi[s3.col[keep]])
                Cn = Cn.toarray()
                for m in ("sig", "any"):                      # an empty row exports start 0, length 0
                    lo[m] = np.where(hi[m] < 0, 0, lo[m])
                st = plan.export_table(c, "CF_START", ax, n)
                end = st + plan.export_table(c, "CF_LEN", ax, n) - 1
                same = (lo["sig"] == lo["any"]) & (hi["sig"] == hi["any"])
                assert same.mean() > 0.99
                assert np.array_equal(st[same], lo["sig"][same]) and np.array_equal(end[same], hi["sig"][same])
                assert (lo["any"] <= st).all() and (st <= lo["sig"]).all()
                assert (hi["sig"] <= end).all() and (end <= hi["any"]).all()
                _weights_match(plan, c, "CF", ax, n, Cn, rel=1e-12)


@pytest.mark.parametrize("name", ["tiny_hex", "tiny_disk"])
def test_nonseparable_lenslet_stage_terms(name):
    """Reading R12: the plan's T separable terms reproduce the oracle's literal per-lenslet 2-D lenslet stage,
    sum_tau S^tau_ks (x) S^tau_kt == sum_mu B^{d mu}_ks (x) B^{d mu}_kt diag(M_mu), for every view (fp64 tables)."""
    cfg = make_config(name)
    plan = lfm.Plan(cfg, device=-1)
    cam = build_system(cfg)[0].camera
    T = plan.info(0)["s3_terms"]
    assert T > 1
    n_s, n_t = cfg["cameras"][0]["n_s"], cfg["cameras"][0]["n_t"]
    n_as, n_at = cam.array_planes[0].n, cam.array_planes[1].n

    def table(ax, idx, n_rows, n_src):
        st = plan.export_table(0, "S3F_START", ax, idx)
        ln = plan.export_table(0, "S3F_LEN", ax, idx)
        w = plan.export_table(0, "S3F_W64", ax, idx).reshape(n_rows, -1)
        M = np.zeros((n_rows, n_src))
        for i in range(n_rows):
            M[i, st[i]:st[i] + ln[i]] = w[i, :ln[i]]
        return M

    for ks in range(cam.ks):
        for kt in range(cam.kt):
            got = sum(np.kron(table(1, kt * T + t, n_t, n_at), table(0, ks * T + t, n_s, n_as)) for t in range(T))
            ref = sum(np.kron(Bt.toarray(), Bs.toarray()) * m.ravel()[None, :] for Bs, Bt, m in cam.S3_2d[ks, kt])
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (ks, kt)
