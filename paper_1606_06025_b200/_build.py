"""Build (nvcc, sm_100a) and load the in-tree CUDA library ``csrc/libgc.so``."""
from __future__ import annotations

import ctypes
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_PATH = os.path.join(CSRC, "libgc.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-diag-suppress", "128"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/gc_api.cu (+ headers) into csrc/libgc.so for sm_100a."""
    srcs = _sources()
    if (not force and os.path.exists(LIB_PATH)
            and all(os.path.getmtime(LIB_PATH) >= os.path.getmtime(s) for s in srcs)):
        return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", tmp, os.path.join(CSRC, "gc_api.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def load() -> ctypes.CDLL:
    """Load libgc.so (building it if stale).  Raises if it cannot be built or loaded:
    the product path has no CPU fallback.  GC_LIB_PATH overrides the path (debug builds)."""
    if os.environ.get("GC_LIB_PATH"):
        return ctypes.CDLL(os.environ["GC_LIB_PATH"])
    try:
        path = build()
    except (OSError, subprocess.CalledProcessError) as e:  # pragma: no cover
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"paper_1606_06025_b200: CUDA library missing and build failed: {e}")
        path = LIB_PATH
    return ctypes.CDLL(path)
