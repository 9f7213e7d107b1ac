"""Write tests/golden/oracle_256_four_camera.json: fp64 ORACLE outputs of the 256^3 four-camera config (BASELINE
configs[3]) at sampled detector pixels and voxels, for the GPU parity test at that size (tests/test_gpu_fullsize.py).

Calls only oracle/ (and the seeded input recipes in workloads/): per camera c, y = A_c x on the flame phantom and
g = A_c^T r_c with r_c = uniform_vector(n_pix, 1 + c), both computed in full by the oracle's matrix-free fp64 path
(literal transposes, no symmetry trick); stored are max |y|, max |g| (the denominators of reading Z24) and the values
at 192 seeded random indices plus the 16 largest entries of each.  The oracle takes ~10 minutes per camera here
(one process per camera).

    python tools/gen_golden_256.py
"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "oracle_256_four_camera.json")
CONFIG = "256^3 four-camera"


def _samples(v, seed, n_rand=192, n_top=16):
    import numpy as np
    rng = np.random.default_rng(seed)
    idx = set(int(i) for i in rng.integers(0, v.size, n_rand))
    idx |= set(int(i) for i in np.argsort(np.abs(v))[-n_top:])
    idx = sorted(idx)
    return {"max_abs": float(np.abs(v).max()), "idx": idx, "val": [float(v[i]) for i in idx]}


def one_camera(c):
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle.system import SystemOperator
    from workloads import flame_volume, make_config, uniform_vector
    cfg = make_config(CONFIG)
    with threadpool_limits(limits=1):
        t0 = time.time()
        x = flame_volume(cfg["volume"]).astype(np.float64)
        op = SystemOperator(cfg["volume"], cfg["cameras"][c])
        t1 = time.time()
        y = op.forward(x)
        r = uniform_vector(op.n_pix, 1 + c).astype(np.float64)
        g = op.adjoint(r)
        t2 = time.time()
    print("camera %d: build %.0f s, forward + adjoint %.0f s" % (c, t1 - t0, t2 - t1), flush=True)
    return {"camera": c, "pose": list(cfg["cameras"][c]["R"]), "y": _samples(y, 100 + c), "g": _samples(g, 200 + c)}


def main():
    from workloads import make_config
    n_cam = len(make_config(CONFIG)["cameras"])
    with mp.get_context("fork").Pool(n_cam) as pool:
        cams = pool.map(one_camera, range(n_cam))
    doc = {"what": "fp64 oracle samples of the 256^3 four-camera config (BASELINE.json configs[3])",
           "written_by": "tools/gen_golden_256.py (calls oracle/ only)",
           "inputs": "x = workloads.flame_volume(volume); r_c = workloads.uniform_vector(n_pix, 1 + c)",
           "metric": "reading Z24: max |gpu - oracle| over the samples / max |oracle| over all outputs",
           "cameras": cams}
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(doc, f)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
