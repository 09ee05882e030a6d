"""Build the sm_100a shared library in-tree (no torch JIT cache involved).

    python -m paper_2506_17626_b200.build

Produces paper_2506_17626_b200/libfeatlsq_b200.so from csrc/*.cu with
`nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -shared`.
The C-ABI it exports is include/featlsq_b200.h.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
# FEATLSQ_LIB: alternative output path for tuning builds (default in-tree)
LIB = os.environ.get("FEATLSQ_LIB") or os.path.join(HERE, "libfeatlsq_b200.so")
SOURCES = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HEADERS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
    os.path.join(ROOT, "include", "featlsq_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--cudart", "static",
         "-Xptxas", "-v", "-diag-suppress", "177"]
# tuning experiments only (e.g. FEATLSQ_NVCC_EXTRA="-DWY_STAGES64=4")
EXTRA = os.environ.get("FEATLSQ_NVCC_EXTRA", "").split()


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a extension")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "_build", os.path.basename(LIB))
    os.makedirs(bdir, exist_ok=True)
    log = []
    for src in SOURCES:
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *ARCH, *FLAGS, *EXTRA, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log.append(res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stderr}")
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "--cudart", "static", "-o", tmp, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    with open(os.path.join(bdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
