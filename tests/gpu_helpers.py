"""Shared helpers for the -m gpu parity tests: run the CUDA path through the C-ABI binding and
the fp64 oracle on the same seeded inputs."""
import numpy as np
import torch

from oracle.system import build_system
from workloads import make_config

_cache = {}


def setup(name):
    key = name if isinstance(name, str) else name["name"]
    if key in _cache:
        return _cache[key]
    from paper_1812_03358_b200 import lfm
    cfg = make_config(name) if isinstance(name, str) else name
    plan = lfm.Plan(cfg, device=0)
    ops = build_system(cfg)
    ws = plan.workspace()
    _cache[key] = (cfg, plan, ops, ws)
    return cfg, plan, ops, ws


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32), device="cuda:0")


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def max_rel(gpu, ref):
    """Reading Z24: max_i |y_hat_i - y_i| / max_i |y_i|."""
    ref = np.asarray(ref, np.float64).ravel()
    gpu = np.asarray(gpu, np.float64).ravel()
    return np.abs(gpu - ref).max() / max(np.abs(ref).max(), 1e-300)


TOL = 1e-5  # north star: max relative error of the fp32 path against the fp64 oracle
