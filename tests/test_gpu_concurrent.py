"""GPU: the concurrent per-camera pair (parallel.ConcurrentPair on CUDA streams, private volumes summed by
lfm_vol_accumulate) equals the sequential pair, and both equal the fp64 oracle within the parity bar."""
import numpy as np
import pytest
import torch

from oracle.system import build_system
from tests.gpu_helpers import TOL, dev, host, max_rel
from workloads import make_config, uniform_vector, uniform_volume

pytestmark = pytest.mark.gpu


def test_vol_accumulate():
    from paper_1812_03358_b200 import lfm
    a = torch.rand(100003, device="cuda:0")
    b = torch.rand(100003, device="cuda:0")
    ref = (a + b).cpu()
    lfm.vol_accumulate(a, b)
    torch.cuda.synchronize()
    assert torch.equal(b.cpu(), ref)
    # 4-byte offset views: the scalar kernel instead of the float4 one, same result
    a1, b1 = a[1:], b[1:]
    ref1 = (a1 + b1).cpu()
    lfm.vol_accumulate(a1, b1)
    torch.cuda.synchronize()
    assert torch.equal(b1.cpu(), ref1)
    with pytest.raises(lfm.LfmError):
        lfm.vol_accumulate(a, a)


@pytest.mark.parametrize("name", ["small_two", "tiny_multi"])
def test_concurrent_pair_matches_sequential(name):
    from paper_1812_03358_b200 import lfm
    from paper_1812_03358_b200.parallel import ConcurrentPair, PairRunner
    cfg = make_config(name)
    plan = lfm.Plan(cfg, device=0)
    ops = build_system(cfg)
    items = [(c, 0, cam["n_t"], 0, cam["n_s"]) for c, cam in enumerate(cfg["cameras"])]
    x = dev(uniform_volume(cfg["volume"], 0)).reshape(-1)
    rs = [dev(uniform_vector(op.n_pix, 1 + c)) for c, op in enumerate(ops)]
    n_vox = ops[0].n_vox
    ws0 = plan.workspace()
    ys_a = [torch.empty(op.n_pix, device="cuda:0") for op in ops]
    g_a = torch.empty(n_vox, device="cuda:0")
    PairRunner(items, lambda c, w, xv, y: lfm.A_forward_window(plan, c, *w, xv, y, ws0),
               lambda c, w, r, g, acc: lfm.A_adjoint_window(plan, c, *w, r, g, ws0, accumulate=acc),
               lambda g: g.zero_()).pair(x, ys_a, rs, g_a)
    streams = [torch.cuda.Stream() for _ in items]
    wss = [plan.workspace() for _ in items]
    private = [None] + [torch.full((n_vox,), float("nan"), device="cuda:0") for _ in items[1:]]
    main = torch.cuda.current_stream()
    start = torch.cuda.Event()
    start.record(main)

    def run(i, fn):
        streams[i].wait_event(start)
        with torch.cuda.stream(streams[i]):
            fn()

    ys_b = [torch.full((op.n_pix,), float("nan"), device="cuda:0") for op in ops]
    g_b = torch.full((n_vox,), float("nan"), device="cuda:0")
    ConcurrentPair(items, lambda i, c, w, xv, y: lfm.A_forward_window(plan, c, *w, xv, y, wss[i]),
                   lambda i, c, w, r, g: lfm.A_adjoint_window(plan, c, *w, r, g, wss[i]),
                   lambda src, dst: lfm.vol_accumulate(src, dst), lambda g: g.zero_(), run,
                   lambda: [main.wait_stream(s) for s in streams], private).pair(x, ys_b, rs, g_b)
    torch.cuda.synchronize()
    for a, b in zip(ys_a, ys_b):
        assert torch.equal(a, b)
    assert max_rel(host(g_b), host(g_a).astype(np.float64)) <= 1e-6
    ref = sum(op.adjoint(host(r).astype(np.float64)) for op, r in zip(ops, rs))
    assert max_rel(host(g_b), ref) <= TOL
