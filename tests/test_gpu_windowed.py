"""The tcgen05 t pass (band_u) in its slice-pair tile mode (u_mode 1: 2 voxel rows x 64 slices per tile, used
when nz % 64 == 0) under the two conditions the other suites do not reach:

* an odd number of voxel rows (the last tile holds one voxel row), checked element by element against the
  fp64 oracle (tolerance 1e-5, reading Z24);
* detector-row windows (lfm_A_forward_rows / lfm_A_adjoint_rows, the multi-GPU sharding calls) at 64^3 and
  128^3 with ragged cuts: the rows of a windowed forward equal those of the full forward, and the windowed
  adjoints over a partition sum to the full adjoint (no oracle needed: both sides are the CUDA path, so the
  tolerance is the fp32 re-association bound 1e-5 of max |.|).
The plan is built with the default kernel choice (band_u for both t passes, band_v for both s passes)."""
import numpy as np
import pytest
import torch

from oracle.system import build_system
from tests.gpu_helpers import TOL, dev, host, max_rel
from workloads import make_config, uniform_vector, uniform_volume

pytestmark = pytest.mark.gpu


def _plan(cfg):
    from paper_1812_03358_b200 import lfm
    plan = lfm.Plan(cfg, device=0)
    for c in range(plan.n_cam):
        assert plan.infos[c]["kind_stage"] == [8, 8], "band_u not chosen"
    return plan


def test_odd_ny_slice_pair_tiles():
    from paper_1812_03358_b200 import lfm
    cfg = make_config("odd_ny")
    assert cfg["volume"]["ny"] % 2 == 1 and cfg["volume"]["nz"] % 64 == 0
    plan = _plan(cfg)
    ws = plan.workspace()
    ops = build_system(cfg)
    x = uniform_volume(cfg["volume"], 0)
    for c, op in enumerate(ops):
        y = torch.empty(op.n_pix, device="cuda:0")
        lfm.A_forward(plan, c, dev(x), y, ws)
        assert max_rel(host(y), op.forward(x.astype(np.float64))) <= TOL
        r = uniform_vector(op.n_pix, 1 + c)
        g = torch.full((op.n_vox,), float("nan"), device="cuda:0")
        lfm.A_adjoint(plan, c, dev(r), g, ws)
        ref = op.adjoint(r.astype(np.float64))
        got = host(g)
        assert np.isfinite(got).all()
        assert max_rel(got, ref) <= TOL
        # the last voxel row (the half-filled tile) explicitly
        nx, ny, nz = cfg["volume"]["nx"], cfg["volume"]["ny"], cfg["volume"]["nz"]
        last = got.reshape(nz, ny, nx)[:, ny - 1, :]
        assert max_rel(last, ref.reshape(nz, ny, nx)[:, ny - 1, :]) <= TOL * np.abs(ref).max() / np.abs(
            ref.reshape(nz, ny, nx)[:, ny - 1, :]).max()


@pytest.mark.parametrize("name", ["64^3 single", "128^3 two-camera"])
def test_row_windows_partition(name):
    from paper_1812_03358_b200 import lfm
    cfg = make_config(name)
    plan = _plan(cfg)
    ws = plan.workspace()
    x = torch.as_tensor(uniform_volume(cfg["volume"], 0), device="cuda:0").reshape(-1)
    for c in range(plan.n_cam):
        inf = plan.infos[c]
        n_t = inf["n_t"]
        y_full = torch.empty(inf["n_pix"], device="cuda:0")
        lfm.A_forward(plan, c, x, y_full, ws)
        yf = host(y_full).reshape(n_t, -1)
        cuts = [0, 5, n_t // 4 + 37, n_t // 2 + 1, (3 * n_t) // 4 - 3, n_t]   # ragged, not tile multiples
        y = torch.full((inf["n_pix"],), float("nan"), device="cuda:0")
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            lfm.A_forward_rows(plan, c, r0, r1, x, y, ws)
            got = host(y).reshape(n_t, -1)[r0:r1]
            assert np.abs(got - yf[r0:r1]).max() <= TOL * np.abs(yf).max()
        r = torch.as_tensor(uniform_vector(inf["n_pix"], 1 + c), device="cuda:0")
        g_full = torch.empty(inf["n_vox"], device="cuda:0")
        lfm.A_adjoint(plan, c, r, g_full, ws)
        g = torch.empty(inf["n_vox"], device="cuda:0")
        for i, (r0, r1) in enumerate(zip(cuts[:-1], cuts[1:])):
            lfm.A_adjoint_rows(plan, c, r0, r1, r, g, ws, accumulate=i > 0)
        gf = host(g_full)
        assert max_rel(host(g), gf) <= TOL


def _col_cuts(n_s):
    # ragged, multiples of 4 (band_v's TMA column alignment) but not of the 256-column tiles
    return [0, n_s // 6 - (n_s // 6) % 4 + 4, n_s // 2 + 4, (3 * n_s) // 4 + 8, n_s]


@pytest.mark.parametrize("name", ["64^3 single", "128^3 two-camera"])
def test_column_and_tile_windows_partition(name):
    """Column windows (the multi-GPU shards of DESIGN.md §7) and 2-D tiles: windowed forwards reproduce the full
    forward on their window; windowed adjoints over a partition sum to the full adjoint.  A 256-column window and
    a quarter of the rows leave most SMs idle, so band_u's forward runs split-K there (partials summed in order)."""
    from paper_1812_03358_b200 import lfm
    cfg = make_config(name)
    plan = _plan(cfg)
    ws = plan.workspace()
    x = torch.as_tensor(uniform_volume(cfg["volume"], 0), device="cuda:0").reshape(-1)
    for c in range(plan.n_cam):
        inf = plan.infos[c]
        n_t, n_s = inf["n_t"], inf["n_s"]
        y_full = torch.empty(inf["n_pix"], device="cuda:0")
        lfm.A_forward(plan, c, x, y_full, ws)
        yf = host(y_full).reshape(n_t, n_s)
        r = torch.as_tensor(uniform_vector(inf["n_pix"], 1 + c), device="cuda:0")
        g_full = torch.empty(inf["n_vox"], device="cuda:0")
        lfm.A_adjoint(plan, c, r, g_full, ws)
        gf = host(g_full)
        ccuts = _col_cuts(n_s)
        windows = [(0, n_t, a, b) for a, b in zip(ccuts[:-1], ccuts[1:])]
        windows_2d = [(r0, r1, c0, c1) for r0, r1 in ((0, n_t // 2 + 3), (n_t // 2 + 3, n_t))
                      for c0, c1 in ((0, n_s // 4 + 12), (n_s // 4 + 12, n_s))]
        windows_small = [(0, n_t // 4, 0, n_s), (0, n_t, 256, 512)]     # split-K shapes
        for wins in (windows, windows_2d):
            y = torch.full((inf["n_pix"],), float("nan"), device="cuda:0")
            g = torch.empty(inf["n_vox"], device="cuda:0")
            for i, (r0, r1, c0, c1) in enumerate(wins):
                lfm.A_forward_window(plan, c, r0, r1, c0, c1, x, y, ws)
                got = host(y).reshape(n_t, n_s)[r0:r1, c0:c1]
                assert np.abs(got - yf[r0:r1, c0:c1]).max() <= TOL * np.abs(yf).max(), (c, r0, r1, c0, c1)
                lfm.A_adjoint_window(plan, c, r0, r1, c0, c1, r, g, ws, accumulate=i > 0)
            assert max_rel(host(g), gf) <= TOL, (c, wins)
        for r0, r1, c0, c1 in windows_small:
            y = torch.full((inf["n_pix"],), float("nan"), device="cuda:0")
            lfm.A_forward_window(plan, c, r0, r1, c0, c1, x, y, ws)
            got = host(y).reshape(n_t, n_s)[r0:r1, c0:c1]
            assert np.abs(got - yf[r0:r1, c0:c1]).max() <= TOL * np.abs(yf).max(), (c, r0, r1, c0, c1)


@pytest.mark.parametrize("name", ["small_two", "small_hex"])
@pytest.mark.parametrize("path", [0, 1])
def test_windows_vs_oracle(path, name):
    """Window entry points against the fp64 oracle: A^T P y with P the window mask, on both evaluation orders
    (the per-view path applies a column window by masking y); small_hex sums T > 1 lenslet-stage terms."""
    from paper_1812_03358_b200 import lfm
    cfg = make_config(name)
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    ops = build_system(cfg)
    x = uniform_volume(cfg["volume"], 0)
    for c, op in enumerate(ops):
        n_t, n_s = cfg["cameras"][c]["n_t"], cfg["cameras"][c]["n_s"]
        r = uniform_vector(op.n_pix, 1).reshape(n_t, n_s)
        yref = op.forward(x.astype(np.float64)).reshape(n_t, n_s)
        for r0, r1, c0, c1 in ((0, n_t, 0, 24), (0, n_t, 24, n_s), (5, 40, 8, 52)):
            y = torch.full((op.n_pix,), float("nan"), device="cuda:0")
            lfm.A_forward_window(plan, c, r0, r1, c0, c1, dev(x), y, ws, path=path)
            got = host(y).reshape(n_t, n_s)[r0:r1, c0:c1]
            assert np.abs(got - yref[r0:r1, c0:c1]).max() <= TOL * np.abs(yref).max()
            m = np.zeros_like(r)
            m[r0:r1, c0:c1] = r[r0:r1, c0:c1]
            g = torch.empty(op.n_vox, device="cuda:0")
            lfm.A_adjoint_window(plan, c, r0, r1, c0, c1, dev(r), g, ws, path=path)
            assert max_rel(host(g), op.adjoint(m.ravel().astype(np.float64))) <= TOL
