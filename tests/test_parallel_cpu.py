"""Multi-rank host logic on CPU (gloo, world_size 2, 3 and 4): the partition covers every detector pixel of
every camera exactly once (column tiles, the default, and row tiles), and the all-reduced partial adjoints of the
ranks equal the single-process adjoint; rank-local forward windows equal the corresponding window of the full
forward.  The per-item operators here are the fp64 oracle restricted to a window (tests may use the oracle)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_03358_b200.parallel import ConcurrentPair, PairRunner, shard


@pytest.mark.parametrize("axis", ["cols", "rows"])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("dims", [[(32, 32)], [(32, 32), (32, 32)], [(2048, 2048)] * 2, [(21, 35), (32, 32), (32, 32)],
                                  [(2048, 2048)] * 4])
def test_partition_covers_pixels_once(world, dims, axis):
    seen = [np.zeros(d, int) for d in dims]
    for r in range(world):
        for c, r0, r1, c0, c1 in shard(dims, r, world, axis=axis):
            seen[c][r0:r1, c0:c1] += 1
            if axis == "cols" and 0 < c0:
                assert c0 % 4 == 0
    for s in seen:
        assert (s == 1).all()


def _worker(rank, world, port, out, mode="seq", axis="cols"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.system import build_system
        from workloads import make_config, uniform_vector, uniform_volume
        cfg = make_config("tiny_multi")
        ops = build_system(cfg)
        dims = [(c["n_t"], c["n_s"]) for c in cfg["cameras"]]
        x = uniform_volume(cfg["volume"], 0).astype(np.float64).ravel()
        rs = [uniform_vector(op.n_pix, 1 + c).astype(np.float64) for c, op in enumerate(ops)]

        def fwd_win(c, win, xv, y):
            r0, r1, c0, c1 = win
            full = ops[c].forward(xv).reshape(dims[c])
            y.reshape(dims[c])[r0:r1, c0:c1] = full[r0:r1, c0:c1]

        def adj_win(c, win, r, g, acc):
            r0, r1, c0, c1 = win
            rr = np.zeros(dims[c])
            rr[r0:r1, c0:c1] = r.reshape(dims[c])[r0:r1, c0:c1]
            v = ops[c].adjoint(rr.ravel())
            if acc:
                g += v
            else:
                g[:] = v

        def allreduce(g):
            t = torch.from_numpy(g)
            dist.all_reduce(t)
            g[:] = t.numpy()

        items = shard(dims, rank, world, axis=axis)
        if mode == "seq":
            runner = PairRunner(items, fwd_win, adj_win, lambda g: g.fill(0.0), allreduce)
        else:  # per-item "streams" are plain calls on CPU; private volumes for items >= 1
            private = [None] + [np.zeros(ops[0].n_vox) for _ in items[1:]]
            runner = ConcurrentPair(items, lambda i, c, w, xv, y: fwd_win(c, w, xv, y),
                                    lambda i, c, w, r, tgt: adj_win(c, w, r, tgt, False),
                                    lambda src, dst: dst.__iadd__(src), lambda g: g.fill(0.0),
                                    lambda i, fn: fn(), lambda: None, private, allreduce)
        ys = [np.full(op.n_pix, np.nan) for op in ops]
        g = np.zeros(ops[0].n_vox)
        runner.pair(x, ys, rs, g)
        ref_g = sum(op.adjoint(r) for op, r in zip(ops, rs))
        ok_g = np.abs(g - ref_g).max() <= 1e-12 * np.abs(ref_g).max()
        ok_y = True
        for c, r0, r1, c0, c1 in items:
            full = ops[c].forward(x).reshape(dims[c])
            ok_y &= np.array_equal(ys[c].reshape(dims[c])[r0:r1, c0:c1], full[r0:r1, c0:c1])
        out[rank] = bool(ok_g and ok_y)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,axis", [(2, "cols"), (4, "cols"), (4, "rows")])
@pytest.mark.parametrize("mode", ["seq", "conc"])
def test_gloo_pair_equals_single_process(world, mode, axis):
    port = 29500 + 7 * world + (13 if mode == "conc" else 0) + (50 if axis == "rows" else 0) + os.getpid() % 200
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out, mode, axis), nprocs=world, join=True)
    assert all(out[r] for r in range(world))


def test_concurrent_pair_sums_in_item_order():
    """ConcurrentPair on one process: every item's forward rows, and g = A_0^T r_0 + A_1^T r_1 + ... added
    in item order -- bitwise the sequential PairRunner result."""
    from oracle.system import build_system
    from workloads import make_config, uniform_vector, uniform_volume
    cfg = make_config("tiny_multi")
    ops = build_system(cfg)
    x = uniform_volume(cfg["volume"], 0).astype(np.float64).ravel()
    rs = [uniform_vector(op.n_pix, 1 + c).astype(np.float64) for c, op in enumerate(ops)]
    items = [(c, 0, cam["n_t"], 0, cam["n_s"]) for c, cam in enumerate(cfg["cameras"])]
    assert len(items) >= 2

    def fwd(c, win, xv, y):
        y[:] = ops[c].forward(xv)

    def adj(c, win, r, g, acc):
        v = ops[c].adjoint(r)
        if acc:
            g += v
        else:
            g[:] = v

    ys1 = [np.zeros(op.n_pix) for op in ops]
    g1 = np.zeros(ops[0].n_vox)
    PairRunner(items, fwd, adj, lambda g: g.fill(0.0)).pair(x, ys1, rs, g1)
    order = []
    ys2 = [np.zeros(op.n_pix) for op in ops]
    g2 = np.full(ops[0].n_vox, np.nan)
    private = [None] + [np.full(ops[0].n_vox, np.nan) for _ in items[1:]]
    ConcurrentPair(items, lambda i, c, w, xv, y: fwd(c, w, xv, y),
                   lambda i, c, w, r, tgt: adj(c, w, r, tgt, False),
                   lambda src, dst: (order.append(id(src)), dst.__iadd__(src)), lambda g: g.fill(0.0),
                   lambda i, fn: fn(), lambda: None, private).pair(x, ys2, rs, g2)
    assert order == [id(p) for p in private[1:]]
    assert np.array_equal(g1, g2)
    for a, b in zip(ys1, ys2):
        assert np.array_equal(a, b)
