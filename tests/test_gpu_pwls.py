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
