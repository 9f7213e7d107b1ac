"""GPU parity of the PWLS pieces (stats, gains, gradient, cost, majoriser, FISTA) with the oracle."""
import numpy as np
import pytest
import torch

from oracle import pwls
from tests.gpu_helpers import TOL, dev, host, max_rel, setup
from workloads import uniform_vector, uniform_volume

pytestmark = pytest.mark.gpu


def _problem(name="tiny_multi", seed=0):
    cfg, plan, ops, ws = setup(name)
    rng = np.random.default_rng(seed)
    x_true = uniform_volume(cfg["volume"], 0).astype(np.float64)
    g_true = [1.0, 0.7, 1.9, 1.3][:len(ops)]
    ys = [op.forward(x_true) / g for op, g in zip(ops, g_true)]
    ws_ = [(rng.random(op.n_pix) + 0.5) * (rng.random(op.n_pix) > 0.05) for op in ops]   # 5% dead pixels
    return cfg, plan, ops, ys, ws_, g_true


@pytest.mark.parametrize("path", [0, 1])
def test_stats_gains_grad_cost(path):
    from paper_1812_03358_b200 import lfm
    from paper_1812_03358_b200.recon import PWLS
    cfg, plan, ops, ys, ws_, g_true = _problem()
    beta, nu = 0.02, 0.003
    rec = PWLS(plan, [dev(y) for y in ys], [dev(w) for w in ws_], beta, nu, path=path)
    x = uniform_volume(cfg["volume"], 4).astype(np.float64) * 0.5
    g = rec.gradient(dev(x), with_cost=True)
    ref, Ax, st, gam = pwls.gradient(x, ops, ys, ws_, beta, nu, return_parts=True)
    assert np.allclose(host(rec.stats).reshape(-1, 3), np.array(st), rtol=2e-6)
    assert np.allclose(host(rec.gamma), gam, rtol=2e-6)
    assert max_rel(host(g), ref) <= TOL
    c = host(rec.cost)
    ref_cost = pwls.cost(x, Ax, ys, ws_, gam, beta, nu)
    assert abs(c.sum() - ref_cost) <= 1e-5 * abs(ref_cost)
    # gains recovered exactly at the truth
    rec.gradient(dev(uniform_volume(cfg["volume"], 0)))
    assert np.allclose(host(rec.gamma), g_true, rtol=1e-5)


def test_majoriser():
    cfg, plan, ops, ys, ws_, _ = _problem()
    from paper_1812_03358_b200.recon import PWLS
    rec = PWLS(plan, [dev(y) for y in ys], [dev(w) for w in ws_], 0.05)
    d = host(rec.majoriser())
    ref = pwls.majoriser(ops, ws_, 0.05, (16, 16, 16)).ravel()
    assert max_rel(d, ref) <= TOL


def test_fista_trajectory():
    """FISTA on device vs the oracle FISTA (reading Z18) for 8 iterations: same iterates to 1e-4."""
    from paper_1812_03358_b200.recon import PWLS
    cfg, plan, ops, ys, ws_, _ = _problem()
    beta, nu = 0.01, 0.0
    rec = PWLS(plan, [dev(y) for y in ys], [dev(w) for w in ws_], beta, nu)
    xs_gpu = []
    rec.fista(8, callback=lambda it, x: xs_gpu.append(host(x)))
    xs_ref = []
    pwls.fista(ops, ys, ws_, beta, nu, (16, 16, 16), 8, callback=lambda it, x: xs_ref.append(x.ravel().copy()))
    for a, b in zip(xs_gpu, xs_ref):
        assert max_rel(a, b) <= 1e-4
    assert (xs_gpu[-1] >= 0).all()


def test_nonfinite_cost_status():
    """a non-finite cost is an error -- lfm_pwls_grad returns LFM_E_NONFINITE when the cost is
    requested; without a cost pointer the call stays asynchronous and returns LFM_OK."""
    from paper_1812_03358_b200 import lfm
    from paper_1812_03358_b200.recon import PWLS
    cfg, plan, ops, ys, ws_, _ = _problem()
    rec = PWLS(plan, [dev(y) for y in ys], [dev(w) for w in ws_], 0.01)
    x = uniform_volume(cfg["volume"], 4).astype(np.float32)
    x[3] = np.nan
    with pytest.raises(lfm.LfmError) as e:
        rec.gradient(dev(x), with_cost=True)
    assert e.value.status == 6
    rec.gradient(dev(x), with_cost=False)   # no cost requested: no check, no error
    torch.cuda.synchronize()
    assert np.isnan(host(rec.grad)).any()


@pytest.mark.parametrize("n", [64, 96])
def test_reg26_vector_and_scalar_footprints_agree(n, monkeypatch):
    """The regulariser gradient (+ cost) with the float4 footprint loads (nx % 4 == 0) and with the scalar loads
    (LFM_R26_SCALAR, read per call) is the same arithmetic on the same values: bit-identical, several blocks in
    every direction and a partial 16-slice z chunk (nz = n - 24)."""
    import torch
    from paper_1812_03358_b200 import lfm
    from workloads import normal_vector
    from workloads.geometry import plenoptic_camera, volume
    cfg = dict(volume=volume(n, 0.4), cameras=[plenoptic_camera(4, 8, 0.04, 2, 2)])
    cfg["volume"]["nz"] = n - 24   # a partial 16-slice chunk
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    nv = plan.infos[0]["n_vox"]
    x = torch.as_tensor(normal_vector(nv, 7), device="cuda:0")
    outs = []
    for scalar in (False, True):
        if scalar:
            monkeypatch.setenv("LFM_R26_SCALAR", "1")
        else:
            monkeypatch.delenv("LFM_R26_SCALAR", raising=False)
        g = torch.empty(nv, device="cuda:0")
        cost = torch.zeros(2, dtype=torch.float64, device="cuda:0")
        lfm.pwls_grad(plan, x, [], [], [], None, 0.05, 0.01, g, ws, cost=cost, cam0=0, cam1=0, include_reg=True)
        torch.cuda.synchronize()
        outs.append((g.cpu(), cost.cpu()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
    # gradient only (the FISTA loop's call): the float4 path sums the neighbours as sliding 3 x 3 plane sums, the
    # scalar one as the literal 26 differences -- the same value up to fp32 summation order
    gs = []
    for scalar in (False, True):
        if scalar:
            monkeypatch.setenv("LFM_R26_SCALAR", "1")
        else:
            monkeypatch.delenv("LFM_R26_SCALAR", raising=False)
        g = torch.empty(nv, device="cuda:0")
        lfm.pwls_grad(plan, x, [], [], [], None, 0.05, 0.01, g, ws, cam0=0, cam1=0, include_reg=True)
        torch.cuda.synchronize()
        gs.append(g.cpu().double())
    assert torch.equal(gs[1], outs[1][0].double())   # the scalar gradient is the same with and without the cost
    assert float((gs[0] - gs[1]).abs().max() / gs[1].abs().max()) <= 1e-6


@pytest.mark.parametrize("name", ["small_two", "small_hex", "128^3 two-camera"])
def test_fused_residual_gradient(name, monkeypatch):
    """lfm_pwls_grad without a cost fuses r = W (A z - gamma y) into the adjoint's column-scaled input split (r never
    stored); with LFM_NO_FUSED_RES the residual kernel writes r first.  Same arithmetic per element, so the two
    gradients are bit-identical; both match the oracle gradient on the small configs."""
    import torch
    from paper_1812_03358_b200 import lfm
    from workloads import make_config, uniform_vector, uniform_volume
    cfg = make_config(name)
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    n = plan.n_cam
    x = torch.as_tensor(uniform_volume(cfg["volume"], 0), device="cuda:0").reshape(-1)
    ys = [torch.as_tensor(uniform_vector(plan.infos[c]["n_pix"], 1 + c), device="cuda:0") for c in range(n)]
    wts = [torch.as_tensor(0.5 + uniform_vector(plan.infos[c]["n_pix"], 7 + c), device="cuda:0") for c in range(n)]
    Axs = [torch.empty(plan.infos[c]["n_pix"], device="cuda:0") for c in range(n)]
    for c in range(n):
        lfm.A_forward(plan, c, x, Axs[c], ws)
    gamma = torch.tensor([1.0, 0.7, 1.3, 0.9][:n], dtype=torch.float64, device="cuda:0")
    gs = []
    for fused in (True, False):
        if fused:
            monkeypatch.delenv("LFM_NO_FUSED_RES", raising=False)
        else:
            monkeypatch.setenv("LFM_NO_FUSED_RES", "1")
        g = torch.empty_like(x)
        lfm.pwls_grad(plan, x, ys, wts, Axs, gamma, 0.01, 0.0, g, ws)
        torch.cuda.synchronize()
        gs.append(g.clone())
    assert torch.equal(gs[0], gs[1])
    assert torch.isfinite(gs[0]).all()


def test_grad_accumulate_contract():
    """LFM_GRAD_ACCUMULATE: a call over no cameras with the regulariser adds R's gradient to grad (no zero fill),
    so grad(cam 0..n) == grad(cameras, no reg) then (+reg, accumulate); with a cost it is rejected."""
    import torch
    from paper_1812_03358_b200 import lfm
    from workloads import make_config, uniform_vector, uniform_volume
    cfg = make_config("small_two")
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    n = plan.n_cam
    x = torch.as_tensor(uniform_volume(cfg["volume"], 0), device="cuda:0").reshape(-1)
    ys = [torch.as_tensor(uniform_vector(plan.infos[c]["n_pix"], 1 + c), device="cuda:0") for c in range(n)]
    wts = [torch.ones(plan.infos[c]["n_pix"], device="cuda:0") for c in range(n)]
    Axs = [torch.empty(plan.infos[c]["n_pix"], device="cuda:0") for c in range(n)]
    for c in range(n):
        lfm.A_forward(plan, c, x, Axs[c], ws)
    gamma = torch.tensor([1.0, 0.8], dtype=torch.float64, device="cuda:0")
    g1 = torch.empty_like(x)
    lfm.pwls_grad(plan, x, ys, wts, Axs, gamma, 0.02, 0.001, g1, ws)
    g2 = torch.empty_like(x)
    lfm.pwls_grad(plan, x, ys, wts, Axs, gamma, 0.02, 0.001, g2, ws, include_reg=False)
    lfm.pwls_grad(plan, x, ys, wts, Axs, gamma, 0.02, 0.001, g2, ws, cam0=0, cam1=0, include_reg=1 | lfm.GRAD_ACCUMULATE)
    torch.cuda.synchronize()
    assert torch.equal(g1, g2)
    cost = torch.zeros(2, dtype=torch.float64, device="cuda:0")
    with pytest.raises(lfm.LfmError):
        lfm.pwls_grad(plan, x, ys, wts, Axs, gamma, 0.02, 0.001, g2, ws, include_reg=1 | lfm.GRAD_ACCUMULATE, cost=cost)
