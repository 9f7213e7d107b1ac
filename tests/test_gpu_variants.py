"""GPU parity of the detector-row entry points (lfm_A_forward_rows / lfm_A_adjoint_rows, the calls the
multi-GPU partition and bench.py use) and of every kernel variant the autotuner may pick for the
streamed t-pass ops, forced one at a time through LFM_FORCE_<op> (so the parity does not depend on
which variant wins the timing on a given box).  Oracle: fp64, element by element, tolerance 1e-5."""
import numpy as np
import pytest
import torch

from oracle.system import build_system
from tests.gpu_helpers import TOL, dev, host, max_rel, setup
from workloads import make_config, uniform_vector, uniform_volume

pytestmark = pytest.mark.gpu


def _masked_rows(r, n_t, r0, r1):
    rr = r.reshape(n_t, -1).copy()
    rr[:r0] = 0.0
    rr[r1:] = 0.0
    return rr.ravel()


@pytest.mark.parametrize("name", ["small_two", "tiny_multi"])
@pytest.mark.parametrize("path", [0, 1])
def test_rows_entry_points(name, path):
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = setup(name)
    x = uniform_volume(cfg["volume"], 0)
    for c, op in enumerate(ops):
        n_t = cfg["cameras"][c]["n_t"]
        cuts = [0, n_t // 3 + 1, (2 * n_t) // 3 - 1, n_t]   # ragged, not multiples of any tile
        yref = op.forward(x.astype(np.float64)).reshape(n_t, -1)
        y = torch.full((op.n_pix,), float("nan"), device="cuda:0")
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            lfm.A_forward_rows(plan, c, r0, r1, dev(x), y, ws, path=path)
            got = host(y).reshape(n_t, -1)[r0:r1]
            assert max_rel(got, yref[r0:r1]) <= TOL * np.abs(yref).max() / np.abs(yref[r0:r1]).max()
        r = uniform_vector(op.n_pix, 1)
        g = torch.empty(op.n_vox, device="cuda:0")
        for i, (r0, r1) in enumerate(zip(cuts[:-1], cuts[1:])):
            lfm.A_adjoint_rows(plan, c, r0, r1, dev(r), g, ws, accumulate=i > 0, path=path)
            if i == 0:
                part = op.adjoint(_masked_rows(r, n_t, r0, r1).astype(np.float64))
                assert max_rel(host(g), part) <= TOL
        assert max_rel(host(g), op.adjoint(r.astype(np.float64))) <= TOL


# ts,tt,nt,nb,stage,kind,stages[,mseg rows]: band_m (MSEG L2 gather) kind=3 with unroll and MSEG group rows ;
# band_f (flat MSEG entries) kind=5 with unroll ; band_u (tcgen05 3xTF32, 128-row tiles) kind=8, stages = drain
# group ; sep: MODE variants (stage 1 = staged U, 0 = U from L2)
VARIANTS = {
    "band_m_128x16_u4": "128,16,128,1,0,3,4",
    "band_m_128x32_u8": "128,32,256,1,0,3,8",
    "band_m_64x16_u8": "64,16,64,1,0,3,8",
    "band_m_32x32_u4": "32,32,64,1,0,3,4",
    "band_m8_128x32_u4": "128,32,128,1,0,3,4,8",
    "band_m8_64x32_u8": "64,32,64,1,0,3,8,8",
    "band_f_128x16_u1": "128,16,128,1,0,5,1",
    "band_f_64x32_u2": "64,32,128,1,0,5,2",
    "band_u_g4": "256,128,384,1,0,8,4",
    "band_u_g1": "256,128,384,1,0,8,1",
    "band_u_g8": "256,128,384,1,0,8,8",
    "sep_64x32_l2": "64,32,128,1,0",
    "sep_32x32_staged": "32,32,64,1,1",
}


@pytest.mark.parametrize("op_name", ["adj_c1", "fwd_c2"])
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_forced_t_pass_variants(op_name, variant, monkeypatch):
    from paper_1812_03358_b200 import lfm
    cfg = make_config("small_two")
    monkeypatch.setenv("LFM_FORCE_" + op_name, VARIANTS[variant])
    monkeypatch.setenv("LFM_FWD_SPLIT", "1")
    monkeypatch.delenv("LFM_TUNE_FILE", raising=False)
    try:
        plan = lfm.Plan(cfg, device=0)
    except lfm.LfmError as e:  # the variant's staged footprint does not fit this op's shared memory
        assert "not applicable" in str(e) or "too large" in str(e), str(e)
        pytest.skip(str(e))
    ws = plan.workspace()
    ops = build_system(cfg)
    x = uniform_volume(cfg["volume"], 0)
    for c, op in enumerate(ops):
        n_t = cfg["cameras"][c]["n_t"]
        y = torch.empty(op.n_pix, device="cuda:0")
        lfm.A_forward(plan, c, dev(x), y, ws, path=1)
        assert max_rel(host(y), op.forward(x.astype(np.float64))) <= TOL, (variant, c)
        r = uniform_vector(op.n_pix, 1)
        g = torch.empty(op.n_vox, device="cuda:0")
        lfm.A_adjoint(plan, c, dev(r), g, ws, path=1)
        assert max_rel(host(g), op.adjoint(r.astype(np.float64))) <= TOL, (variant, c)
        # windowed source rows (adjoint row sharding) and output rows (forward row sharding)
        r0, r1 = n_t // 4 + 1, (3 * n_t) // 4
        lfm.A_adjoint_rows(plan, c, r0, r1, dev(r), g, ws, path=1)
        assert max_rel(host(g), op.adjoint(_masked_rows(r, n_t, r0, r1).astype(np.float64))) <= TOL, (variant, c)
        y.fill_(float("nan"))
        lfm.A_forward_rows(plan, c, r0, r1, dev(x), y, ws, path=1)
        yref = op.forward(x.astype(np.float64)).reshape(n_t, -1)
        assert max_rel(host(y).reshape(n_t, -1)[r0:r1], yref[r0:r1]) <= TOL * np.abs(yref).max() / np.abs(yref[r0:r1]).max()


@pytest.mark.parametrize("name", ["small_two", "tiny_multi", "tiny_dirac"])
@pytest.mark.parametrize("transposed", ["0", "1", "2", "3"])
def test_s_pass_orders(name, transposed, monkeypatch):
    """The three s-pass forms of the two-pass collapsed path (0: direct sep kernel, 1: transpose + band_m/band_f
    with transposed output, 2: the direct s-pass kernels of spass.cuh, 3: the tcgen05 s passes of band_v.cuh), forced, against the oracle: forward,
    adjoint and their row-range forms."""
    from paper_1812_03358_b200 import lfm
    cfg = make_config(name)
    monkeypatch.setenv("LFM_FWD_SPLIT", "1")
    monkeypatch.setenv("LFM_FWD_T", transposed)
    monkeypatch.setenv("LFM_ADJ_T", transposed)
    monkeypatch.delenv("LFM_TUNE_FILE", raising=False)
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    ops = build_system(cfg)
    x = uniform_volume(cfg["volume"], 0)
    for c, op in enumerate(ops):
        n_t = cfg["cameras"][c]["n_t"]
        y = torch.empty(op.n_pix, device="cuda:0")
        lfm.A_forward(plan, c, dev(x), y, ws, path=1)
        assert max_rel(host(y), op.forward(x.astype(np.float64))) <= TOL, (name, c)
        r = uniform_vector(op.n_pix, 1)
        g = torch.full((op.n_vox,), 0.5, device="cuda:0")
        lfm.A_adjoint(plan, c, dev(r), g, ws, accumulate=True, path=1)
        ref = 0.5 + op.adjoint(r.astype(np.float64))
        assert max_rel(host(g), ref) <= TOL, (name, c)
        r0, r1 = n_t // 3, n_t - 3
        lfm.A_adjoint_rows(plan, c, r0, r1, dev(r), g, ws, path=1)
        assert max_rel(host(g), op.adjoint(_masked_rows(r, n_t, r0, r1).astype(np.float64))) <= TOL, (name, c)


@pytest.mark.parametrize("name", ["small_two", "small_hex"])
@pytest.mark.parametrize("bk", ["16", "32", "64"])
def test_band_v_adjoint_block_width(name, bk, monkeypatch):
    """band_v's adjoint s pass with K blocks of 16 / 32 / 64 detector columns (LFM_VBK_A; 32 and 64 have 2xFP16
    images, so the fp16 Z of the t pass feeds them directly, 64 with 128-byte rows) against the oracle, also on a
    column window (the K-window instance)."""
    from paper_1812_03358_b200 import lfm
    cfg = make_config(name)
    monkeypatch.setenv("LFM_VBK_A", bk)
    monkeypatch.delenv("LFM_TUNE_FILE", raising=False)
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    ops = build_system(cfg)
    for c, op in enumerate(ops):
        r = uniform_vector(op.n_pix, 1)
        g = torch.empty(op.n_vox, device="cuda:0")
        lfm.A_adjoint(plan, c, dev(r), g, ws, path=1)
        assert max_rel(host(g), op.adjoint(r.astype(np.float64))) <= TOL, (name, bk, c)
        n_s, n_t = cfg["cameras"][c]["n_s"], cfg["cameras"][c]["n_t"]
        c0, c1 = 8, n_s - 5
        lfm.A_adjoint_window(plan, c, 0, n_t, c0, c1, dev(r), g, ws, path=1)
        rm = r.reshape(n_t, n_s).copy()
        rm[:, :c0] = 0
        rm[:, c1:] = 0
        assert max_rel(host(g), op.adjoint(rm.reshape(-1).astype(np.float64))) <= TOL, (name, bk, c, "window")


def test_stage_entry_points():
    """lfm_A_stage runs the forward / adjoint t pass alone on the workspace intermediate (one band_u launch, plus the
    ordered split-K sum on small outputs, as in A_forward; the adjoint's 2xFP16 form also splits its input):
    FWD_T after a forward reproduces that forward's y bit for bit; bad stage ids and NULLs fail."""
    from paper_1812_03358_b200 import lfm
    cfg, plan, ops, ws = setup("small_two")
    x = dev(uniform_volume(cfg["volume"], 0))
    for c, op in enumerate(ops):
        y = torch.empty(op.n_pix, device="cuda:0")
        try:
            lfm.A_forward(plan, c, x, y, ws, path=1)
            y2 = torch.full_like(y, float("nan"))
            lfm.A_stage(plan, c, lfm.STAGE_FWD_T, None, y2, ws)
        except lfm.LfmError as e:
            assert "two-pass" in str(e)
            continue
        assert lfm.last_launch_count() in (1, 2)     # band_u, plus the ordered chunk sum when it splits K
        assert torch.equal(y, y2)
        lfm.A_stage(plan, c, lfm.STAGE_ADJ_T, dev(uniform_vector(op.n_pix, 1)), None, ws)
        # band_u (3xTF32); column-scaled fp16 split + band_u (2xFP16, fp16 Z); maxima + fp16 split + band_u
        assert lfm.last_launch_count() in (1, 2, 3)
        with pytest.raises(lfm.LfmError):
            lfm.A_stage(plan, c, 7, None, y2, ws)
        with pytest.raises(lfm.LfmError):
            lfm.A_stage(plan, c, lfm.STAGE_ADJ_T, None, None, ws)
