"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the partition covers every detector row of
every camera exactly once, and the all-reduced partial adjoints of the ranks equal the single-process
adjoint; rank-local forward rows equal the corresponding rows of the full forward.  The per-item
operators here are the fp64 oracle restricted to rows (tests may use the oracle)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_03358_b200.parallel import PairRunner, shard


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("rows", [[32], [32, 32], [2048, 2048], [21, 32, 32], [2048] * 4])
def test_partition_covers_rows_once(world, rows):
    seen = [np.zeros(n, int) for n in rows]
    for r in range(world):
        for c, r0, r1 in shard(rows, r, world):
            seen[c][r0:r1] += 1
    for s in seen:
        assert (s == 1).all()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.system import build_system
        from workloads import make_config, uniform_vector, uniform_volume
        cfg = make_config("tiny_multi")
        ops = build_system(cfg)
        n_rows = [c["n_t"] for c in cfg["cameras"]]
        x = uniform_volume(cfg["volume"], 0).astype(np.float64).ravel()
        rs = [uniform_vector(op.n_pix, 1 + c).astype(np.float64) for c, op in enumerate(ops)]

        def fwd_rows(c, r0, r1, xv, y):
            full = ops[c].forward(xv).reshape(n_rows[c], -1)
            y.reshape(n_rows[c], -1)[r0:r1] = full[r0:r1]

        def adj_rows(c, r0, r1, r, g, acc):
            rr = r.reshape(n_rows[c], -1).copy()
            rr[:r0] = 0.0
            rr[r1:] = 0.0
            v = ops[c].adjoint(rr.ravel())
            if acc:
                g += v
            else:
                g[:] = v

        def allreduce(g):
            t = torch.from_numpy(g)
            dist.all_reduce(t)
            g[:] = t.numpy()

        items = shard(n_rows, rank, world)
        runner = PairRunner(items, fwd_rows, adj_rows, lambda g: g.fill(0.0), allreduce)
        ys = [np.full(op.n_pix, np.nan) for op in ops]
        g = np.zeros(ops[0].n_vox)
        runner.pair(x, ys, rs, g)
        ref_g = sum(op.adjoint(r) for op, r in zip(ops, rs))
        ok_g = np.abs(g - ref_g).max() <= 1e-12 * np.abs(ref_g).max()
        ok_y = True
        for c, r0, r1 in items:
            full = ops[c].forward(x).reshape(n_rows[c], -1)
            ok_y &= np.array_equal(ys[c].reshape(n_rows[c], -1)[r0:r1], full[r0:r1])
        out[rank] = bool(ok_g and ok_y)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_pair_equals_single_process(world):
    port = 29500 + 7 * world + os.getpid() % 200
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))
