"""NEXT-3 angular-basis study (sec,angular P:477-522) at a size the oracle renders in seconds: the GPU
renderings of the pillbox and Dirac models at K = 1, 2, 4 per axis match the oracle's (1e-5), and the
scale-fitted NSD against the finest Dirac rendering (reading R6) reproduces the paper's qualitative claims:
the pillbox model is more accurate than the Dirac one at coarse angular sampling, and both converge with K."""
import numpy as np
import pytest
import torch

from oracle.system import build_system
from tests.gpu_helpers import TOL, host, max_rel
from workloads import flame_volume
from workloads.geometry import DIRAC, PILLBOX, plenoptic_camera, volume

pytestmark = pytest.mark.gpu


def _nsd(y, ref):
    a = float(y @ ref / (y @ y))
    return float(np.sum((a * y - ref) ** 2) / np.sum(ref ** 2))


def test_angular_study_small():
    from paper_1812_03358_b200 import lfm
    vol = volume(32, 0.4)
    x = flame_volume(vol).astype(np.float32)
    xd = torch.as_tensor(x, device="cuda:0").reshape(-1)

    def gpu(basis, k):
        cfg = dict(name="a", volume=vol, cameras=[plenoptic_camera(8, 8, 0.04, k, 2, basis=basis)])
        plan = lfm.Plan(cfg, device=0)
        ws = plan.workspace()
        y = torch.empty(plan.infos[0]["n_pix"], device="cuda:0")
        lfm.A_forward(plan, 0, xd, y, ws)
        return host(y), build_system(cfg)[0]

    ref, _ = gpu(DIRAC, 16)
    nsd = {}
    for k in (1, 2, 4):
        for basis in (PILLBOX, DIRAC):
            y, op = gpu(basis, k)
            assert max_rel(y, op.forward(x.astype(np.float64))) <= TOL
            nsd[basis, k] = _nsd(y, ref)
    assert nsd[PILLBOX, 1] < 0.5 * nsd[DIRAC, 1]
    assert nsd[PILLBOX, 2] < 0.5 * nsd[DIRAC, 2]
    for basis in (PILLBOX, DIRAC):
        assert nsd[basis, 4] < nsd[basis, 2] < nsd[basis, 1]
