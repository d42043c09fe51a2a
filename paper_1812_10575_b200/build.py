"""Build librbm.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

    python -m paper_1812_10575_b200.build [--force]

Seven translation units (the C ABI + one engine unit per (dtype, d)) compile
in parallel and link into paper_1812_10575_b200/librbm.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "librbm.so")
BUILD = os.path.join(PKG, "_build")
UNITS = ["rbm_api.cu"] + [f"rbm_engines_{t}_d{d}.cu" for t in ("f32", "f64") for d in (1, 2, 3)]
HEADERS = ["rbm_device.cuh", "rbm_kernels.cuh", "rbm_host.cuh", "rbm_nccl.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", f"-I{os.path.join(ROOT, 'include')}"]


def _sources():
    return ([os.path.join(CSRC, u) for u in UNITS] + [os.path.join(CSRC, h) for h in HEADERS]
            + [os.path.join(ROOT, "include", "rbm.h")])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile the units in parallel and link `out` (default librbm.so);
    `defines` (e.g. ["RBM_EXPERIMENT=1"]) build a design-experiment variant."""
    lib = out or LIB
    if not force and not defines and not stale():
        return LIB
    bdir = BUILD if not defines else BUILD + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(bdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def compile_unit(u):
        obj = os.path.join(bdir, u.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *dflags, "-Xptxas", "-v", "-c", os.path.join(CSRC, u), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(bdir, u + ".ptxas.log"), "w") as f:
            f.write(r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {u}:\n{r.stderr[-4000:]}")
        return obj

    with cf.ThreadPoolExecutor(len(UNITS)) as ex:
        objs = list(ex.map(compile_unit, UNITS))
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, lib)
    if verbose:
        print("built", lib)
    return lib


CHECKED = os.path.join(PKG, "librbm_checked.so")


def build_checked(force: bool = False) -> str:
    """librbm_checked.so: the same library with index bounds asserted in the
    kernels (-DRBM_CHECKED=1; the memory-safety tier, tests/test_checked_gpu.py)."""
    if not force and os.path.exists(CHECKED) and os.path.getmtime(CHECKED) >= max(
            os.path.getmtime(p) for p in _sources()):
        return CHECKED
    return build(force=True, out=CHECKED, defines=["RBM_CHECKED=1"])


if __name__ == "__main__":
    # python -m paper_1812_10575_b200.build [--force] [-DNAME=V ... -o out.so]
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    out = sys.argv[sys.argv.index("-o") + 1] if "-o" in sys.argv else None
    build(force="--force" in sys.argv, verbose=True, out=out, defines=defs)
