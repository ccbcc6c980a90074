"""Build liblmdtw_b200.so in-tree with nvcc for sm_100a.

    python paper_2008_02734_b200/build.py [--force]   (a script: importing the
    package needs a current library, building must not)

The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "liblmdtw_b200.so")
OBJDIR = os.path.join(HERE, "_build")
SOURCES = ["kernels.cu", "window.cu", "engine.cu"]
HEADERS = [os.path.join(CSRC, "lmdtw_internal.h"), os.path.join(CSRC, "sqrt64_fast.cuh"), os.path.join(INCLUDE, "lmdtw_b200.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: ptxas otherwise fuses mul.rn.f32x2 + add.rn.f32x2 into FFMA2,
# breaking bit parity; -ffp-contract=off: same rule for host-side path_cost.
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
         "-Xptxas", "-warn-spills", "-I", CSRC, "-I", INCLUDE] + os.environ.get("LMDTW_NVCC_EXTRA", "").split()


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    objs, procs = [], []
    # kernels.cu is compiled twice (fp32 / fp64 strip engines) so the two
    # halves build in parallel
    units = [("kernels.cu", "kernels_f32.o", ["-DLMDTW_TU=32"]), ("kernels.cu", "kernels_f64.o", ["-DLMDTW_TU=64"])]
    units += [(src, src.replace(".cu", ".o"), []) for src in SOURCES if src != "kernels.cu"]
    for src, obj, defs in units:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJDIR, obj)
        objs.append(o)
        if force or _stale(o, [s] + HEADERS):
            cmd = [NVCC] + ARCH + FLAGS + defs + ["-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{out.decode(errors='replace')}")
        if verbose and out:
            print(out.decode(errors="replace"))
    if force or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {r.stdout}{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
