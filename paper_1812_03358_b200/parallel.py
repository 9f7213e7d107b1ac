"""Multi-GPU partition of an A + A^T pair: one process per GPU, NCCL over NVLink.

Work items are (camera, detector window [r0, r1) x [c0, c1)).  Cameras are dealt round-robin over the ranks; with
more ranks than cameras every camera's detector is split into contiguous tiles -- by default along the detector
columns s, the axis the collapsed operator's s passes act on column by column, so a column shard shrinks every
kernel of the pair (band_v items, band_u tiles; DESIGN.md §7 has the per-rank timings), or along the rows t.
Forward projection needs no communication (x is replicated; each rank produces its window of y_c).  The adjoint
of each rank covers only its window (A_c^T P_window y_c); the partial volumes are summed by ONE all-reduce of
n_vox fp32 values -- the only data-path collective.  Orchestration only: the per-item operators are injected
(the C-ABI calls on a GPU; any implementation in the CPU tests).
"""


def _split(n, k, align):
    """k contiguous tiles of [0, n) with inner edges on multiples of `align` (empty tiles dropped)."""
    edges = [0] + [min(n, (n * i // k + align // 2) // align * align) for i in range(1, k)] + [n]
    return [(a, b) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def shard(dims, rank, world, axis="cols", align=4):
    """Items (camera, r0, r1, c0, c1) of `rank`; dims[c] = (n_t, n_s) of camera c.  axis "cols": tiles of
    columns whose inner edges are multiples of `align` (band_v moves 16-byte column groups); "rows": tiles of
    rows."""
    n_cam = len(dims)
    if world <= n_cam:
        return [(c, 0, dims[c][0], 0, dims[c][1]) for c in range(n_cam) if c % world == rank]
    per = world // n_cam
    extra = world - per * n_cam                     # the first `extra` cameras get one more tile
    c, slot = 0, rank
    while c < n_cam:
        tiles = per + (1 if c < extra else 0)
        if slot < tiles:
            n_t, n_s = dims[c]
            if axis == "rows":
                parts = _split(n_t, tiles, 1)
                return [(c, parts[slot][0], parts[slot][1], 0, n_s)] if slot < len(parts) else []
            parts = _split(n_s, tiles, align)
            return [(c, 0, n_t, parts[slot][0], parts[slot][1])] if slot < len(parts) else []
        slot -= tiles
        c += 1
    return []


class PairRunner:
    """One A+A^T pair of this rank.

    forward_win(c, win, x, y_c) -> writes the window win = (r0, r1, c0, c1) of y_c
    adjoint_win(c, win, r_c, g, accumulate) -> g (+)= A_c^T P_win r_c
    zero(g); allreduce(g) (None on one rank)
    """

    def __init__(self, items, forward_win, adjoint_win, zero, allreduce=None):
        self.items = items
        self.forward_win = forward_win
        self.adjoint_win = adjoint_win
        self.zero = zero
        self.allreduce = allreduce

    def forward(self, x, ys):
        for c, *win in self.items:
            self.forward_win(c, tuple(win), x, ys[c])

    def adjoint(self, rs, g):
        first = True
        for c, *win in self.items:
            self.adjoint_win(c, tuple(win), rs[c], g, not first)
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

    def __init__(self, items, forward_win, adjoint_win, accumulate, zero, run, join, private, allreduce=None):
        self.items = items
        self.forward_win = forward_win        # (i, c, win, x, y)
        self.adjoint_win = adjoint_win        # (i, c, win, r, g_target)   overwrite
        self.accumulate = accumulate          # (src, dst)                 dst += src
        self.zero = zero
        self.run = run                        # (i, fn)
        self.join = join                      # ()
        self.private = private                # private[i] for i >= 1: volume buffers
        self.allreduce = allreduce

    def compute(self, x, ys, rs, g):
        """Everything but the all-reduce (what a per-rank CUDA graph captures)."""
        for i, (c, *win) in enumerate(self.items):
            tgt = g if i == 0 else self.private[i]
            w = tuple(win)
            self.run(i, lambda i=i, c=c, w=w, tgt=tgt: (self.forward_win(i, c, w, x, ys[c]),
                                                        self.adjoint_win(i, c, w, rs[c], tgt)))
        self.join()
        if not self.items:
            self.zero(g)
        for i in range(1, len(self.items)):
            self.accumulate(self.private[i], g)

    def pair(self, x, ys, rs, g):
        self.compute(x, ys, rs, g)
        if self.allreduce is not None:
            self.allreduce(g)
