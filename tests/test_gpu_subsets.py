"""View-subset operators and the ordered-subsets PWLS gradient (sec,subset P:360-388; reading Z19/R5) on the
GPU through the C ABI, element by element against the fp64 oracle (tolerance 1e-5, reading Z24)."""
import numpy as np
import pytest
import torch

from oracle import pwls
from oracle.system import build_system
from tests.gpu_helpers import TOL, dev, host, max_rel
from workloads import make_config, normal_vector, uniform_vector, uniform_volume

pytestmark = pytest.mark.gpu

_plans = {}


def _plan(name, M):
    from paper_1812_03358_b200 import lfm
    key = (name, M)
    if key not in _plans:
        cfg = make_config(name)
        plan = lfm.Plan(cfg, device=0, n_subsets=M)
        _plans[key] = (cfg, plan, build_system(cfg), plan.workspace())
    return _plans[key]


@pytest.mark.parametrize("name,M", [("tiny_k4", 4), ("tiny_k4", 3), ("small_two", 4), ("tiny_multi", 2),
                                    ("tiny_dirac", 2)])
def test_subset_forward_adjoint(name, M):
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _plan(name, M)
    x = uniform_volume(cfg["volume"], 0)
    for c, op in enumerate(ops):
        cam = op.camera
        r = normal_vector(op.n_pix, 3)
        for m in range(M):
            S = pwls.subset_views(cam.ks, cam.kt, M, m)
            s = cam.ks * cam.kt / len(S)
            y = torch.empty(op.n_pix, device="cuda:0")
            lfm.A_forward_subset(plan, c, m, dev(x), y, ws)
            assert max_rel(host(y), s * op.forward(x.astype(np.float64), S)) <= TOL, (name, c, m)
            g = torch.full((op.n_vox,), 0.25, device="cuda:0")
            lfm.A_adjoint_subset(plan, c, m, dev(r), g, ws, accumulate=True)
            assert max_rel(host(g), 0.25 + s * op.adjoint(r.astype(np.float64), S)) <= TOL, (name, c, m)


def test_subset_gradient_matches_oracle():
    from paper_1812_03358_b200.recon import PWLS
    cfg, plan, ops, ws = _plan("tiny_multi", 2)
    x = uniform_volume(cfg["volume"], 0)
    ys = [uniform_vector(op.n_pix, 1 + c) for c, op in enumerate(ops)]
    wts = [(0.5 + uniform_vector(op.n_pix, 5 + c)) for c, op in enumerate(ops)]
    rec = PWLS(plan, [dev(y) for y in ys], [dev(w) for w in wts], 0.02, 0.05)
    for m in range(2):
        g = host(rec.gradient(dev(x), subset=m))
        ref = pwls.gradient_subset(x.astype(np.float64), ops, [y.astype(np.float64) for y in ys],
                                   [w.astype(np.float64) for w in wts], 0.02, 0.05, 2, m)
        assert max_rel(g, ref) <= TOL


def test_ordered_subsets_fista_trajectory():
    from paper_1812_03358_b200.recon import PWLS
    from workloads import flame_volume
    cfg, plan, ops, ws = _plan("small_two", 4)
    x_true = flame_volume(cfg["volume"]).astype(np.float64)
    ys = [op.forward(x_true) / g for op, g in zip(ops, [1.0, 0.7])]
    wts = [np.ones(op.n_pix) for op in ops]
    d_ref = pwls.majoriser(ops, wts, 0.0, (32, 32, 32))
    beta = 0.01 * float(np.median(d_ref))
    rec = PWLS(plan, [dev(y) for y in ys], [dev(w) for w in wts], beta, 0.0)
    xs_gpu = []
    rec.fista(6, callback=lambda it, x: xs_gpu.append(host(x)), subsets=True)
    xs_ref = []
    pwls.fista(ops, ys, wts, beta, 0.0, (32, 32, 32), 6, n_subsets=4,
               callback=lambda it, x: xs_ref.append(x.ravel().copy()))
    for a, b in zip(xs_gpu, xs_ref):
        assert max_rel(a, b) <= 1e-4


def test_subset_errors():
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = _plan("tiny_k4", 4)
    x = dev(uniform_volume(cfg["volume"], 0))
    y = torch.empty(ops[0].n_pix, device="cuda:0")
    with pytest.raises(lfm.LfmError):
        lfm.A_forward_subset(plan, 0, 4, x, y, ws)
    with pytest.raises(lfm.LfmError):
        lfm.A_forward_subset(plan, 0, -1, x, y, ws)
    cfg2, plan2, ops2, ws2 = _plan("tiny_k4", 0)
    with pytest.raises(lfm.LfmError):
        lfm.A_forward_subset(plan2, 0, 0, x, y, ws2)
    with pytest.raises(lfm.LfmError):  # more subsets than views
        lfm.Plan(make_config("tiny"), device=0, n_subsets=5)
