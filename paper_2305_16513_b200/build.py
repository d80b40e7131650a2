"""In-tree build of the CUDA library libss.so (sm_100a) and the synthetic-input
generator libsynth.so.  Invoked by __graft_entry__.build() and by tests."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libss.so")
SOURCES = ["api.cu", "slide1d.cu", "generic.cu", "pool2d.cu", "affine.cu", "conv_tc.cu", "backward.cu", "dilated.cu", "conv2d.cu", "conv2d_backward.cu", "conv_mc.cu", "conv2d_tile.cu", "maxbwd.cu", "fgrad_tc.cu", "mc_fgrad.cu"]
HEADERS = ["ss_device.cuh", "ss_internal.h"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# IEEE arithmetic: no fast-math, no FTZ, IEEE div/sqrt, no FMA contraction
# beyond the explicit __fmaf_rn calls.
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--ftz=false",
         "--prec-div=true", "--prec-sqrt=true", "--fmad=false", "-Xptxas", "-v"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_libss(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "ss.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = [NVCC, *ARCH, *FLAGS, "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for s, p in procs:
        out = p.communicate()[0].decode()
        if verbose:
            print(out)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}:\n{out}")
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build_libss(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
