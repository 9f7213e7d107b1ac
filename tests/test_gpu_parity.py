"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Tolerance (north star): max_i |y_gpu - y_oracle| / max_i |y_oracle| <= 1e-5 (reading Z24).
Inputs: x ~ U[0,1) seed 0, y ~ U[0,1) seed 1, N(0,1) seeds 2/3 for adjoint tests.
"""
import numpy as np
import pytest
import torch

from tests.gpu_helpers import TOL, dev, host, max_rel, setup
from workloads import make_config, normal_vector, uniform_vector, uniform_volume

pytestmark = pytest.mark.gpu

SMALL = ["tiny", "tiny_k4", "tiny_single", "tiny_yaw15", "tiny_multi", "tiny_dirac", "tiny_turn", "small_two", "ragged",
         "tiny_hex", "tiny_disk", "small_hex"]
PATHS = [0, 1]  # PER_VIEW, COLLAPSED


def _ragged_config():
    from workloads.geometry import plenoptic_camera, pose_yaw_pitch, single_camera
    cam = plenoptic_camera(5, 7, 0.05, 3, 2, pose=pose_yaw_pitch(12.0, -7.0))
    cam.update(nl_t=3, n_t=21, k_t=2)
    return dict(name="ragged", volume=dict(nx=19, ny=17, nz=13, dx=0.45, dy=0.4, dz=0.35),
                cameras=[cam, single_camera(23, 0.05, 3, pose=pose_yaw_pitch(-20.0, 10.0))])


def _setup(name):
    return setup(_ragged_config() if name == "ragged" else name)


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("path", PATHS)
def test_forward_parity(name, path):
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _setup(name)
    x = uniform_volume(cfg["volume"], 0)
    xd = dev(x)
    for c, op in enumerate(ops):
        y = torch.empty(op.n_pix, device="cuda:0")
        lfm.A_forward(plan, c, xd, y, ws, path=path)
        ref = op.forward(x.astype(np.float64))
        assert max_rel(host(y), ref) <= TOL, (name, c, path)


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("path", PATHS)
def test_adjoint_parity(name, path):
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _setup(name)
    for c, op in enumerate(ops):
        r = uniform_vector(op.n_pix, 1)
        g = torch.empty(op.n_vox, device="cuda:0")
        lfm.A_adjoint(plan, c, dev(r), g, ws, path=path)
        ref = op.adjoint(r.astype(np.float64))
        assert max_rel(host(g), ref) <= TOL, (name, c, path)


@pytest.mark.parametrize("name", ["tiny_yaw15", "small_two", "ragged"])
def test_adjoint_dot_fp32(name):
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _setup(name)
    for c, op in enumerate(ops):
        for path in PATHS:
            x = dev(normal_vector(op.n_vox, 2))
            r = dev(normal_vector(op.n_pix, 3))
            y = torch.empty(op.n_pix, device="cuda:0")
            g = torch.empty(op.n_vox, device="cuda:0")
            lfm.A_forward(plan, c, x, y, ws, path=path)
            lfm.A_adjoint(plan, c, r, g, ws, path=path)
            lhs = float((y.double() * r.double()).sum())
            rhs = float((x.double() * g.double()).sum())
            assert abs(lhs - rhs) / (float(y.double().norm()) * float(r.double().norm())) <= 1e-5


def test_adjoint_accumulate():
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _setup("tiny_yaw15")
    op = ops[0]
    r = dev(uniform_vector(op.n_pix, 1))
    base = dev(uniform_vector(op.n_vox, 7))
    g = base.clone()
    lfm.A_adjoint(plan, 0, r, g, ws, accumulate=True)
    g2 = torch.empty_like(g)
    lfm.A_adjoint(plan, 0, r, g2, ws, accumulate=False)
    assert torch.allclose(g, base + g2, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("name", ["tiny_yaw15", "ragged", "small_two", "tiny_turn"])
def test_vol_rotate_parity(name):
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _setup(name)
    x = uniform_volume(cfg["volume"], 0)
    for c, op in enumerate(ops):
        out = torch.empty(op.n_vox, device="cuda:0")
        lfm.vol_rotate(plan, c, lfm.FWD, dev(x), out, ws)
        assert max_rel(host(out), op.rot.forward(x.astype(np.float64))) <= TOL
        lfm.vol_rotate(plan, c, lfm.ADJ, dev(x), out, ws)
        assert max_rel(host(out), op.rot.adjoint(x.astype(np.float64))) <= TOL


def _xport_ref(op, dst_kind, src_kind, n, src):
    """Oracle transport for all views: dst_k = (1/V^p) B^{pq}_k src_k, literal matrices."""
    from oracle.transport import basis_volume
    cam = op.camera
    K = cam.ks * cam.kt
    out = []
    for kt in range(cam.kt):
        for ks in range(cam.ks):
            s = src[kt * cam.ks + ks]
            if (dst_kind, src_kind) == ("a", "q") or (dst_kind, src_kind) == ("d", "q"):
                dst = cam.array_planes if dst_kind == "a" else cam.det_planes
                V = basis_volume(dst[0], cam.d0[0]) * basis_volume(dst[1], cam.d0[1])
                out.append(cam.S1[1][kt][n] @ s @ cam.S1[0][ks][n].T / V)
            elif src_kind in ("a", "d") and dst_kind == "q":
                q = cam.slice_planes
                V = basis_volume(q[0][n], cam.d0[0]) * basis_volume(q[1][n], cam.d0[1])
                # B^{qp} = (B^{pq})^T, evaluated literally as a transpose here
                out.append(cam.S1[1][kt][n].T @ s @ cam.S1[0][ks][n] / V)
            elif (dst_kind, src_kind) == ("d", "a"):
                V = basis_volume(cam.lenslet_planes[0][0], cam.d0[0]) * basis_volume(cam.lenslet_planes[1][0], cam.d0[1])
                if cam.nonsep:   # literal per-lenslet 2-D masks (R12/R13)
                    out.append(sum(Bt @ (m * s) @ Bs.T for Bs, Bt, m in cam.S3_2d[ks, kt]) / V)
                else:
                    out.append(cam.S3[1][kt] @ s @ cam.S3[0][ks].T / V)
            elif (dst_kind, src_kind) == ("a", "d"):
                V = basis_volume(cam.array_planes[0], cam.d0[0]) * basis_volume(cam.array_planes[1], cam.d0[1])
                if cam.nonsep:
                    out.append(sum(m * (Bt.T @ s @ Bs) for Bs, Bt, m in cam.S3_2d[ks, kt]) / V)
                else:
                    out.append(cam.S3[1][kt].T @ s @ cam.S3[0][ks] / V)
    return np.stack(out)


@pytest.mark.parametrize("name", ["tiny", "tiny_single", "ragged", "tiny_hex"])
def test_lf_transport_parity(name):
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _setup(name)
    for c, op in enumerate(ops):
        cam = op.camera
        inf = plan.infos[c]
        nz, K = inf["nz"], inf["n_views"]
        A, D = inf["plane_array"], inf["plane_detector"]
        dims = {"q": (op.camera.ny, op.camera.nx), "d": (inf["n_t"], inf["n_s"])}
        if inf["type"] == 1:
            dims["a"] = (inf["n_at"], inf["n_as"])
            pairs = [("a", "q"), ("q", "a"), ("d", "a"), ("a", "d")]
        else:
            pairs = [("d", "q"), ("q", "d")]
        ids = {"a": A, "d": D}
        for n in (0, nz // 2, nz - 1):
            for dst_kind, src_kind in pairs:
                src = uniform_vector(K * dims[src_kind][0] * dims[src_kind][1], 5).reshape(K, *dims[src_kind])
                out = torch.empty(K * dims[dst_kind][0] * dims[dst_kind][1], device="cuda:0")
                lfm.lf_transport(plan, c, ids.get(dst_kind, n), ids.get(src_kind, n), dev(src), out, ws)
                ref = _xport_ref(op, dst_kind, src_kind, n, src.astype(np.float64))
                assert max_rel(host(out), ref) <= TOL, (name, c, dst_kind, src_kind, n)


def test_lf_transport_symmetry_scaling():
    """(V^q/V^p) lf_transport(q,p) is the adjoint of lf_transport(p,q)."""
    from paper_1812_03358_b200 import lfm
    from oracle.transport import basis_volume
    cfg, plan, ops, ws = _setup("tiny")
    op = ops[0]
    cam = op.camera
    inf = plan.infos[0]
    K, A, D = inf["n_views"], inf["plane_array"], inf["plane_detector"]
    na, nd = inf["n_as"] * inf["n_at"], inf["n_s"] * inf["n_t"]
    fa = dev(normal_vector(K * na, 2))
    fd = dev(normal_vector(K * nd, 3))
    out_d = torch.empty(K * nd, device="cuda:0")
    out_a = torch.empty(K * na, device="cuda:0")
    lfm.lf_transport(plan, 0, D, A, fa, out_d, ws)
    lfm.lf_transport(plan, 0, A, D, fd, out_a, ws)
    Va = basis_volume(cam.array_planes[0], cam.d0[0]) * basis_volume(cam.array_planes[1], cam.d0[1])
    Vmu = basis_volume(cam.lenslet_planes[0][0], cam.d0[0]) * basis_volume(cam.lenslet_planes[1][0], cam.d0[1])
    lhs = float((out_d.double() * fd.double()).sum())
    rhs = float((fa.double() * out_a.double()).sum()) * Va / Vmu
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


def test_paths_agree_and_deterministic():
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _setup("small_two")
    x = dev(uniform_volume(cfg["volume"], 0))
    for c, op in enumerate(ops):
        ys = []
        for path in PATHS + [1]:
            y = torch.empty(op.n_pix, device="cuda:0")
            lfm.A_forward(plan, c, x, y, ws, path=path)
            ys.append(y)
        assert torch.equal(ys[1], ys[2])           # bitwise repeatable (no atomics)
        assert max_rel(host(ys[0]), host(ys[1])) <= TOL


def test_zero_input_and_errors():
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _setup("tiny_yaw15")
    op = ops[0]
    y = torch.full((op.n_pix,), 7.0, device="cuda:0")
    lfm.A_forward(plan, 0, torch.zeros(op.n_vox, device="cuda:0"), y, ws)
    assert float(y.abs().max()) == 0.0
    with pytest.raises(lfm.LfmError) as e:
        lfm.lf_transport(plan, 0, 0, 1, y, y, ws)       # slice -> slice unsupported
    assert e.value.status == 4
    small = torch.empty(16, dtype=torch.uint8, device="cuda:0")
    with pytest.raises(lfm.LfmError) as e:
        lfm.A_forward(plan, 0, torch.zeros(op.n_vox, device="cuda:0"), y, small)
    assert e.value.status == 1
    with pytest.raises(lfm.LfmError):
        lfm.A_forward(plan, 5, torch.zeros(op.n_vox, device="cuda:0"), y, ws)


@pytest.mark.parametrize("n_lens,dynamic", [(5, False), (5, True), (7, True)])
def test_collapsed_f16_column_strips(n_lens, dynamic):
    """The 2xFP16 collapsed path on detectors whose width is a multiple of 8 but not of 16 (40 and 56 columns: the
    column-scaled split's last 16-column strip is half empty, band_u's last 256-column tile ragged) against the
    oracle; `dynamic`: detector columns scaled by 10^(-6 .. 0) and voxel rows by 10^(-4 .. 0), so the per-column
    (adjoint input) and per-row (x^r) fp16 scales differ by orders of magnitude across the data."""
    from paper_1812_03358_b200 import lfm
    from oracle.system import build_system
    from workloads.geometry import plenoptic_camera, pose_yaw, volume
    cfg = dict(volume=volume(16, 0.4), cameras=[plenoptic_camera(n_lens, 8, 0.04, 2, 2),
                                                plenoptic_camera(n_lens, 8, 0.04, 2, 2, pose=pose_yaw(20.0))])
    plan = lfm.Plan(cfg, device=0)
    assert plan.infos[0]["f16_stage"] == [1, 1], plan.infos[0]["f16_stage"]
    ws = plan.workspace()
    ops = build_system(cfg)
    x = uniform_volume(cfg["volume"], 0)
    if dynamic:
        x = (x * (10.0 ** np.linspace(-4, 0, x.shape[1]))[None, :, None]).astype(np.float32)
    for c, op in enumerate(ops):
        n_s = cfg["cameras"][c]["n_s"]
        y = torch.empty(op.n_pix, device="cuda:0")
        lfm.A_forward(plan, c, dev(x).reshape(-1), y, ws, path=1)
        assert max_rel(host(y), op.forward(x.astype(np.float64).ravel())) <= TOL, (n_lens, dynamic, c, "forward")
        r = uniform_vector(op.n_pix, 1).reshape(-1, n_s)
        if dynamic:
            r = (r * 10.0 ** np.linspace(-6, 0, n_s)[None, :]).astype(np.float32)
        r = r.ravel()
        g = torch.empty(op.n_vox, device="cuda:0")
        lfm.A_adjoint(plan, c, dev(r), g, ws, path=1)
        assert max_rel(host(g), op.adjoint(r.astype(np.float64))) <= TOL, (n_lens, dynamic, c, "adjoint")


def test_collapsed_tall_detector():
    """A detector taller than the column-scaled split keeps in registers (2112 > 16 x 128 rows: the strip's extra
    rows take the split's second pass) and wider than 8 band_u column tiles, on the collapsed path, against the
    oracle (single-lens camera, 16^3 volume, pixel pitch matched to the voxels' image)."""
    from paper_1812_03358_b200 import lfm
    from oracle.system import build_system
    from workloads.geometry import single_camera, volume
    cfg = dict(volume=volume(16, 0.4), cameras=[single_camera(2112, 0.004, 2)])
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    op = build_system(cfg)[0]
    r = uniform_vector(op.n_pix, 1)
    g = torch.empty(op.n_vox, device="cuda:0")
    lfm.A_adjoint(plan, 0, dev(r), g, ws, path=1)
    assert max_rel(host(g), op.adjoint(r.astype(np.float64))) <= TOL
    x = uniform_volume(cfg["volume"], 0)
    y = torch.empty(op.n_pix, device="cuda:0")
    lfm.A_forward(plan, 0, dev(x).reshape(-1), y, ws, path=1)
    assert max_rel(host(y), op.forward(x.astype(np.float64).ravel())) <= TOL
    assert plan.infos[0]["f16_stage"] == [1, 1], plan.infos[0]["f16_stage"]   # the 2xFP16 tcgen05 path ran
