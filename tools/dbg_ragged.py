"""Debug helper: adjoint parity of one config under forced s-pass modes (LFM_ADJ_T / LFM_FWD_T)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.system import build_system
from paper_1812_03358_b200 import lfm
from workloads import make_config, uniform_vector, uniform_volume
name = sys.argv[1] if len(sys.argv) > 1 else "ragged"
if name == "ragged":
    sys.path.insert(0, ".")
    from tests.test_gpu_parity import _ragged_config
    cfg = _ragged_config()
else:
    cfg = make_config(name)
ops = build_system(cfg)
for mode in ([m for m in os.environ.get("MODES", "0,1,2,N").split(",")]):
    mode = None if mode == "N" else mode
    if mode is None:
        os.environ.pop("LFM_ADJ_T", None); os.environ.pop("LFM_FWD_T", None)
    else:
        os.environ["LFM_ADJ_T"] = mode; os.environ["LFM_FWD_T"] = mode
    plan = lfm.Plan(cfg, device=0); ws = plan.workspace()
    for c, op in enumerate(ops):
        r = uniform_vector(op.n_pix, 1)
        g = torch.empty(op.n_vox, device="cuda:0")
        lfm.A_adjoint(plan, c, torch.as_tensor(r, device="cuda:0"), g, ws, path=1)
        ref = op.adjoint(r.astype(np.float64))
        x = uniform_volume(cfg["volume"], 0)
        y = torch.empty(op.n_pix, device="cuda:0")
        lfm.A_forward(plan, c, torch.as_tensor(x, device="cuda:0").ravel(), y, ws, path=1)
        yr = op.forward(x.astype(np.float64))
        gg = g.cpu().numpy()
        if os.environ.get("DIAG"):
            v = cfg["volume"]; sh = (v["nz"], v["ny"], v["nx"])
            G = gg.reshape(sh); R = ref.reshape(sh)
            a = (G * R).sum() / (R * R).sum()
            print("  fit scale %.4f corr %.4f" % (a, np.corrcoef(G.ravel(), R.ravel())[0, 1]))
            for nm, T in [("flip z", R[::-1]), ("flip y", R[:, ::-1]), ("flip x", R[:, :, ::-1])]:
                print("  corr with", nm, "%.4f" % np.corrcoef(G.ravel(), T.ravel())[0, 1])
            print("  per-slice max |G|", np.abs(G).max(axis=(1, 2))[:6], " |R|", np.abs(R).max(axis=(1, 2))[:6])
        print("mode", mode, "cam", c, "adj err %.3e" % (np.abs(gg - ref).max() / np.abs(ref).max()),
              "fwd err %.3e" % (np.abs(y.cpu().numpy() - yr).max() / np.abs(yr).max()), "nonzero", np.count_nonzero(gg),
              plan.infos[c]["kind_stage"][:], flush=True)
