"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (collapsed path,
128^3 two-camera; also the 64^3 single-camera config), element by element against the fp64
oracle.  At 256^3 four-camera (configs[3]: yaw -30/0/+30 and the pitch-30 camera) the oracle takes ~10 minutes
per camera, so its outputs at sampled pixels/voxels (plus their max |.|) are stored by tools/gen_golden_256.py
(a committed script that calls only oracle/) and compared element by element here; properties that hold at any
size (adjoint identity, agreement of the two evaluation orders) are checked as well."""
import json
import os
import numpy as np
import pytest
import torch

from tests.gpu_helpers import TOL, dev, host, max_rel
from workloads import flame_volume, make_config, normal_vector, uniform_vector

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("name,paths", [("64^3 single", (0, 1)), ("128^3 two-camera", (1,))])
def test_full_size_parity(name, paths):
    from oracle.system import SystemOperator
    from paper_1812_03358_b200 import lfm
    cfg = make_config(name)
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    x = flame_volume(cfg["volume"])
    for c, cam in enumerate(cfg["cameras"]):
        op = SystemOperator(cfg["volume"], cam)
        y_ref = op.forward(x.astype(np.float64))
        r = uniform_vector(op.n_pix, 1)
        g_ref = op.adjoint(r.astype(np.float64))
        for path in paths:
            y = torch.empty(op.n_pix, device="cuda:0")
            lfm.A_forward(plan, c, dev(x).reshape(-1), y, ws, path=path)
            assert max_rel(host(y), y_ref) <= TOL, (name, c, path, "forward")
            g = torch.empty(op.n_vox, device="cuda:0")
            lfm.A_adjoint(plan, c, dev(r), g, ws, path=path)
            assert max_rel(host(g), g_ref) <= TOL, (name, c, path, "adjoint")


def test_256_four_camera_properties():
    from paper_1812_03358_b200 import lfm
    cfg = make_config("256^3 four-camera")
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    n_vox = plan.infos[0]["n_vox"]
    x = dev(normal_vector(n_vox, 2))
    xf = dev(flame_volume(cfg["volume"])).reshape(-1)
    for c in range(plan.n_cam):
        n_pix = plan.infos[c]["n_pix"]
        r = dev(normal_vector(n_pix, 3))
        y = torch.empty(n_pix, device="cuda:0")
        g = torch.empty(n_vox, device="cuda:0")
        lfm.A_forward(plan, c, x, y, ws)
        lfm.A_adjoint(plan, c, r, g, ws)
        lhs = float((y.double() * r.double()).sum())
        rhs = float((x.double() * g.double()).sum())
        assert abs(lhs - rhs) / (float(y.double().norm()) * float(r.double().norm())) <= 1e-5
        y1 = torch.empty(n_pix, device="cuda:0")
        y0 = torch.empty(n_pix, device="cuda:0")
        lfm.A_forward(plan, c, xf, y1, ws, path=lfm.COLLAPSED)
        lfm.A_forward(plan, c, xf, y0, ws, path=lfm.PER_VIEW)
        assert max_rel(host(y0), host(y1)) <= TOL


GOLDEN_256 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_256_four_camera.json")


def test_256_four_camera_sampled_oracle_parity():
    from paper_1812_03358_b200 import lfm
    doc = json.load(open(GOLDEN_256))
    cfg = make_config("256^3 four-camera")
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    x = dev(flame_volume(cfg["volume"])).reshape(-1)
    assert len(doc["cameras"]) == plan.n_cam == 4
    for cam in doc["cameras"]:
        c = cam["camera"]
        assert tuple(cam["pose"]) == tuple(cfg["cameras"][c]["R"])
        n_pix, n_vox = plan.infos[c]["n_pix"], plan.infos[c]["n_vox"]
        r = dev(uniform_vector(n_pix, 1 + c))
        for path in (lfm.COLLAPSED, lfm.PER_VIEW):
            y = torch.empty(n_pix, device="cuda:0")
            lfm.A_forward(plan, c, x, y, ws, path=path)
            yy = host(y)
            err = np.abs(yy[cam["y"]["idx"]] - np.array(cam["y"]["val"])).max() / cam["y"]["max_abs"]
            assert err <= TOL, (c, path, "forward", err)
            assert abs(np.abs(yy).max() - cam["y"]["max_abs"]) <= TOL * cam["y"]["max_abs"]
            g = torch.empty(n_vox, device="cuda:0")
            lfm.A_adjoint(plan, c, r, g, ws, path=path)
            gg = host(g)
            err = np.abs(gg[cam["g"]["idx"]] - np.array(cam["g"]["val"])).max() / cam["g"]["max_abs"]
            assert err <= TOL, (c, path, "adjoint", err)
            assert abs(np.abs(gg).max() - cam["g"]["max_abs"]) <= TOL * cam["g"]["max_abs"]


def test_128_hex_properties():
    """NEXT-4 at the metric's scale (hexagonal layout + circular apertures, T = 2 lenslet-stage terms): the per-view
    and collapsed evaluation orders agree element by element, and the fp32 adjoint identity holds (the oracle's
    literal per-lenslet model would take hours at 128 x 146 lenslets; its parity is at tiny/small sizes)."""
    from paper_1812_03358_b200 import lfm
    cfg = make_config("128^3 hex two-camera")
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    n_vox = plan.infos[0]["n_vox"]
    xf = dev(flame_volume(cfg["volume"])).reshape(-1)
    x = dev(normal_vector(n_vox, 2))
    for c in range(plan.n_cam):
        assert plan.infos[c]["s3_terms"] > 1
        n_pix = plan.infos[c]["n_pix"]
        y0 = torch.empty(n_pix, device="cuda:0")
        y1 = torch.empty(n_pix, device="cuda:0")
        lfm.A_forward(plan, c, xf, y0, ws, path=lfm.PER_VIEW)
        lfm.A_forward(plan, c, xf, y1, ws, path=lfm.COLLAPSED)
        assert max_rel(host(y0), host(y1)) <= TOL
        r = dev(normal_vector(n_pix, 3))
        g0 = torch.empty(n_vox, device="cuda:0")
        g1 = torch.empty(n_vox, device="cuda:0")
        lfm.A_adjoint(plan, c, r, g0, ws, path=lfm.PER_VIEW)
        lfm.A_adjoint(plan, c, r, g1, ws, path=lfm.COLLAPSED)
        assert max_rel(host(g0), host(g1)) <= TOL
        lfm.A_forward(plan, c, x, y1, ws)
        lhs = float((y1.double() * r.double()).sum())
        rhs = float((x.double() * g1.double()).sum())
        assert abs(lhs - rhs) / (float(y1.double().norm()) * float(r.double().norm())) <= 1e-5
