"""Build libchemora.so in-tree: nvcc for sm_100a (fp64 kernels, -lineinfo), C-ABI host
runtime compiled by nvcc/g++, the CUDA driver entry points it needs (stream memory ops for the cross-process slab
signalling) are fetched at run time, so the library loads on a GPU-less host.  Run ``python -m paper_1410_1764_b200.build``."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libchemora.so")
OBJ = os.path.join(HERE, "build_obj")
ROOT = os.path.dirname(HERE)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
           "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
# the wave kernels exist in two tilings that must agree bitwise: no implicit FMA
# contraction there (every fma is explicit in the source)
NO_FMAD = {"wave_stage.cu", "wave_tma.cu", "wave_fused3.cu"}
SOURCES = ["wave_stage.cu", "wave_tma.cu", "wave_fused3.cu", "bssn_stage.cu", "bssn_fused.cu", "ghost_init_norms.cu",
           "capi.cpp"]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "chemora.h")]


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    newest = max(os.path.getmtime(d) for d in _deps())
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    cmd = ["nvcc", *ARCH, *NVFLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cpp"):
        cmd = ["nvcc", "-x", "cu", *cmd[1:]]
    if src in NO_FMAD:
        cmd.insert(1, "-fmad=false")
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(OBJ, os.path.basename(src) + ".log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed for {src}")
    if verbose:
        sys.stderr.write(res.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    # always relink (a few seconds): an mtime test would keep a library copied in from
    # elsewhere (e.g. an A/B build) whose timestamp is newer than the objects
    cmd = ["nvcc", *ARCH, "-shared", "-o", OUT + ".tmp", *objs]
    subprocess.check_call(cmd)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
