"""The rotation passes' kernel variants give bit-identical results (eqn,rot,toeplitz P:1186-1198).

`launch_shear` runs a y pass (poses with pitch) on `shear_y_kernel` (a thread walks its line with a sliding window;
LFM_SH_Y_SCALAR=1 selects the scalar `shear_kernel`) and picks the x-pass kernel (`shear_x4_kernel`, 4 consecutive x per thread from float4 windows, or the
scalar `shear_kernel`) and the z chunk per thread from LFM_SH_X4 / LFM_SH_ZC, read once per process; every
variant keeps the same FMA order per output, so vol_rotate (forward and adjoint, store and accumulate) must
agree bit for bit with the scalar kernel.  Each setting runs in its own process.  Parity of the default against
the oracle is in test_gpu_parity.py."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %(root)r)
from paper_1812_03358_b200 import lfm
from workloads import make_config, uniform_volume
out = {}
for name in %(configs)r:
    cfg = make_config(name)
    plan = lfm.Plan(cfg, device=0)
    ws = plan.workspace()
    x = torch.as_tensor(uniform_volume(cfg["volume"], 3), device="cuda:0").reshape(-1).contiguous()
    for cam in range(len(cfg["cameras"])):
        for d in (lfm.FWD, lfm.ADJ):
            y = torch.empty_like(x)
            lfm.vol_rotate(plan, cam, d, x, y, ws)
            z = torch.full_like(x, 0.25)
            lfm.vol_rotate(plan, cam, d, x, z, ws, accumulate=True)
            torch.cuda.synchronize()
            out["%%s_%%d_%%d_s" %% (name, cam, d)] = y.cpu().numpy()
            out["%%s_%%d_%%d_a" %% (name, cam, d)] = z.cpu().numpy()
np.savez(sys.argv[1], **out)
"""

CONFIGS = ["tiny_multi", "tiny_turn", "small_two"]


def _run(tmp_path, env_extra, tag):
    path = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ)
    env.update(env_extra)
    subprocess.run([sys.executable, "-c", SCRIPT % dict(root=ROOT, configs=CONFIGS), path], env=env, check=True,
                   timeout=600)
    return dict(np.load(path))


@pytest.mark.gpu
def test_shear_variants_bit_identical(tmp_path):
    ref = _run(tmp_path, {"LFM_SH_X4": "0", "LFM_SH_ZC": "8", "LFM_SH_Y_SCALAR": "1"}, "scalar")
    assert any(np.abs(v).max() > 0 for v in ref.values())
    for x4, zc in (("1", "16"), ("2", "32"), ("3", "8"), ("4", "16"), ("5", "8")):
        got = _run(tmp_path, {"LFM_SH_X4": x4, "LFM_SH_ZC": zc}, f"x4_{x4}_zc_{zc}")
        for k, v in ref.items():
            assert np.array_equal(got[k], v), (x4, zc, k)
