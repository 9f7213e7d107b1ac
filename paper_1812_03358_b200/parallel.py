"""Multi-GPU partition of an A + A^T pair: one process per GPU, NCCL over NVLink.

Work items are (camera, detector rows [r0, r1)): cameras are dealt round-robin over the ranks; with
more ranks than cameras every camera's detector rows are split into contiguous tiles.  Forward
projection needs no communication (x is replicated; each rank produces its rows of y_c).  The adjoint
of each rank covers only its rows (A_c^T P_rows y_c); the partial volumes are summed by ONE all-reduce
of n_vox fp32 values -- the only data-path collective.  Orchestration only: the per-item operators
are injected (the C-ABI calls on a GPU; any implementation in the CPU tests).
"""


def shard(n_rows, rank, world):
    """Items (camera, r0, r1) of `rank`; n_rows[c] = detector rows of camera c."""
    n_cam = len(n_rows)
    if world <= n_cam:
        return [(c, 0, n_rows[c]) for c in range(n_cam) if c % world == rank]
    per = world // n_cam
    extra = world - per * n_cam                     # the first `extra` cameras get one more tile
    c, slot = 0, rank
    while c < n_cam:
        tiles = per + (1 if c < extra else 0)
        if slot < tiles:
            r0 = n_rows[c] * slot // tiles
            r1 = n_rows[c] * (slot + 1) // tiles
            return [(c, r0, r1)] if r1 > r0 else []
        slot -= tiles
        c += 1
    return []


class PairRunner:
    """One A+A^T pair of this rank.

    forward_rows(c, r0, r1, x, y_c) -> writes rows [r0, r1) of y_c
    adjoint_rows(c, r0, r1, r_c, g, accumulate) -> g (+)= A_c^T P_[r0,r1) r_c
    zero(g); allreduce(g) (None on one rank)
    """

    def __init__(self, items, forward_rows, adjoint_rows, zero, allreduce=None):
        self.items = items
        self.forward_rows = forward_rows
        self.adjoint_rows = adjoint_rows
        self.zero = zero
        self.allreduce = allreduce

    def forward(self, x, ys):
        for c, r0, r1 in self.items:
            self.forward_rows(c, r0, r1, x, ys[c])

    def adjoint(self, rs, g):
        first = True
        for c, r0, r1 in self.items:
            self.adjoint_rows(c, r0, r1, rs[c], g, not first)
            first = False
        if first:
            self.zero(g)
        if self.allreduce is not None:
            self.allreduce(g)

    def pair(self, x, ys, rs, g):
        self.forward(x, ys)
        self.adjoint(rs, g)


class ConcurrentPair:
    """The same pair with every item on its own CUDA stream and workspace (one process per GPU, items of
    this rank only).  Forwards are independent.  Item 0's adjoint writes g; item i > 0 writes a private
    volume g_i; after all items finish, the g_i are added into g in item order (deterministic: the same
    summation order as the sequential PairRunner, g = ((A_0^T r_0) + A_1^T r_1) + ...).

    run(i, fn) runs fn on item i's stream after the previous call's inputs are visible (injected: CUDA
    streams on a GPU, plain calls on CPU); join() makes the main stream wait for every item;
    accumulate(src, dst) adds on the main stream.
    """

    def __init__(self, items, forward_rows, adjoint_rows, accumulate, zero, run, join, private, allreduce=None):
        self.items = items
        self.forward_rows = forward_rows      # (i, c, r0, r1, x, y)
        self.adjoint_rows = adjoint_rows      # (i, c, r0, r1, r, g_target)   overwrite
        self.accumulate = accumulate          # (src, dst)                     dst += src
        self.zero = zero
        self.run = run                        # (i, fn)
        self.join = join                      # ()
        self.private = private                # private[i] for i >= 1: volume buffers
        self.allreduce = allreduce

    def pair(self, x, ys, rs, g):
        for i, (c, r0, r1) in enumerate(self.items):
            tgt = g if i == 0 else self.private[i]
            self.run(i, lambda i=i, c=c, r0=r0, r1=r1, tgt=tgt: (self.forward_rows(i, c, r0, r1, x, ys[c]),
                                                            self.adjoint_rows(i, c, r0, r1, rs[c], tgt)))
        self.join()
        if not self.items:
            self.zero(g)
        for i in range(1, len(self.items)):
            self.accumulate(self.private[i], g)
        if self.allreduce is not None:
            self.allreduce(g)
