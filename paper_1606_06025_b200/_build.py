"""Build (nvcc, sm_100a) and load the in-tree CUDA library ``csrc/libgc.so``.

Every ``csrc/*.cu`` is compiled to an object in parallel (the persistent kernel instances are
split by state-word width into ``inst_*.cu``), then linked into one shared library.
"""
from __future__ import annotations

import ctypes
import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(CSRC, "obj")
LIB_PATH = os.path.join(CSRC, "libgc.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "128"]


def _headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _units():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale(target, deps):
    return not os.path.exists(target) or any(os.path.getmtime(target) < os.path.getmtime(d) for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile csrc/*.cu (+ headers) into csrc/libgc.so for sm_100a.  `defines` (e.g.
    ["GC_NQ=1"]) and `out` build a tuning variant elsewhere (A/B measurements only)."""
    units, headers = _units(), _headers()
    lib_path = out or LIB_PATH
    obj_dir = OBJ if not defines else os.path.join(os.path.dirname(lib_path), "obj_" + "_".join(defines).replace("=", ""))
    if not force and not defines and not _stale(lib_path, units + headers):
        return lib_path
    os.makedirs(obj_dir, exist_ok=True)
    nvcc = _nvcc()

    def compile_unit(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        if force or _stale(obj, [src] + headers):
            tmp = obj + f".tmp{os.getpid()}"
            cmd = [nvcc, *NVCC_FLAGS, *(["-D" + d for d in defines]), *(["-Xptxas=-v"] if verbose else []), "-c", "-o",
                   tmp, src]
            subprocess.check_call(cmd)
            os.replace(tmp, obj)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(units), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(compile_unit, units))
    tmp = lib_path + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, lib_path)
    return lib_path


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
