"""Builds libspmesl.so in-tree (sm_100a only) with nvcc.

    python -m paper_2203_15031_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libspmesl.so")

SOURCES = ["prep.cu", "cd_sweep.cu", "tail.cu", "joint.cu", "gram_full.cu", "screen16.cu", "assemble.cu",
           "api.cu", "multi.cu", "penalty.cpp"]


def _nccl_dirs():
    """The NCCL header (types only: the library is dlopen-ed at run time) and the pip NCCL's
    shared library, if present (the run-time fallback after the process's own libnccl.so.2)."""
    inc, lib = "/usr/include", ""
    try:
        import nvidia.nccl as _nv
        base = list(_nv.__path__)[0]
        if os.path.exists(os.path.join(base, "include", "nccl.h")):
            inc = os.path.join(base, "include")
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            lib = cand
    except Exception:
        pass
    return inc, lib
HEADERS = [os.path.join(CSRC, "spmesl_internal.cuh"), os.path.join(ROOT, "include", "spmesl.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]
_NCCL_INC, _NCCL_LIB = _nccl_dirs()
FLAGS += ["-I", _NCCL_INC, f'-DSPMESL_NCCL_PIP_LIB="{_NCCL_LIB}"']
# (development: extra -D switches for kernel variants, e.g. SPMESL_NVCC_EXTRA="-DSPMESL_SYRK_MIG=4")
FLAGS += os.environ.get("SPMESL_NVCC_EXTRA", "").split()


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    log = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + HEADERS):
            cmd = [NVCC] + ARCH + FLAGS + ["-c", path, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            log.append(r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if force or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt",
                                                                 "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        # every symbol must resolve (no GPU needed to load the library)
        r = subprocess.run(["python3", "-c", f"import ctypes; ctypes.CDLL({LIB!r})"],
                           capture_output=True, text=True)
        if r.returncode != 0:
            os.remove(LIB)
            raise RuntimeError(f"{LIB} does not load:\n{r.stderr}")
    if verbose:
        print("\n".join(x for x in log if x))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
