"""Build liblfm.so in-tree: nvcc for sm_100a (kernels + C ABI), g++ -ffp-contract=off for the fp64 plan.

    python -m paper_1812_03358_b200.build        # or __graft_entry__.build()
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "liblfm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES_CU = ["kernels.cu", "api.cu"]
SOURCES_CPP = ["plan.cpp"]
HEADERS = ["lfm_internal.h", "lfm_kernels.h", "band_u.cuh", "tc_sm100.h", "spass.cuh", "band_v.cuh"]


def _inputs():
    files = [os.path.join(CSRC, f) for f in SOURCES_CU + SOURCES_CPP + HEADERS]
    files.append(os.path.join(ROOT, "include", "lfm.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:3]))
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)


def build(force=False, verbose=False, ptxas_verbose=False):
    if not force and up_to_date():
        return LIB
    bdir = os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    objs = []
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    for f in SOURCES_CPP:
        o = os.path.join(bdir, f + ".o")
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
              "-I/usr/local/cuda/include"] + inc + ["-c", os.path.join(CSRC, f), "-o", o], verbose)
        objs.append(o)
    for f in SOURCES_CU:
        o = os.path.join(bdir, f + ".o")
        extra = ["-Xptxas", "-v"] if ptxas_verbose else []
        extra += os.environ.get("LFM_NVCC_DEFS", "").split()  # experiments only (e.g. -DBAND_U_NO_MMA)
        _run([NVCC, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off"]
             + ARCH + extra + inc + ["-c", os.path.join(CSRC, f), "-o", o], verbose or ptxas_verbose)
        objs.append(o)
    out = os.environ.get("LFM_BUILD_OUT", LIB)  # experiments: build a variant library beside the product one
    tmp = out + ".tmp"
    _run([NVCC, "-shared", "-cudart", "static"] + ARCH + objs + ["-o", tmp], verbose)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="--ptxas" in sys.argv)
    print(LIB)
