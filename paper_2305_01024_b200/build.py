"""Build libftgemm.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2305_01024_b200.build [--verbose]

Each .cu under csrc/ is compiled to an object with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC
and linked into paper_2305_01024_b200/libftgemm.so (static cudart).  Objects are
cached by source / header mtime.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libftgemm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "ftgemm.h")]
    return max(os.path.getmtime(f) for f in files)


def build(verbose: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """defines / out: development variants (e.g. -DFTGEMM_EXP_NO_Y) built to a separate library."""
    global OBJ, LIB
    if defines or out:
        OBJ = os.path.join(HERE, "build_" + "_".join(d.lstrip("-D").lower() for d in defines))
        LIB = out or os.path.join(HERE, "libftgemm_" + "_".join(d[2:].lower().replace("ftgemm_exp_", "")
                                                                 for d in defines) + ".so")
        force = True
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    dep = _deps_mtime()
    objs, changed = [], force or not os.path.exists(LIB)
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), dep):
            cmd = [NVCC, *ARCH, *FLAGS, *defines, "-c", s, "-o", o]
            if verbose:
                cmd += ["-Xptxas", "-v"]
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            changed = True
    if changed or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", LIB, *objs, "-lcublas"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv, defines=defs))
