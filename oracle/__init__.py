"""CPU oracle for round-synchronous SGR colouring (arXiv 1606.06025) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The CUDA product path
(``paper_1606_06025_b200``) never imports it and shares no code with it.

Thin ctypes marshalling over ``oracle.c`` (plain single-threaded C, see its header for the
paper passages each function follows).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

POLICIES = {"higher_id": 0, "lower_id": 1, "degree": 2}


class NoConvergence(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2, single-threaded; no OpenMP, no vector intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        vp = ctypes.c_void_p
        lib.oracle_sgr.argtypes = [ctypes.c_int64, vp, vp, ctypes.c_int, ctypes.c_int64, vp,
                                   ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                   vp, ctypes.c_int64]
        lib.oracle_greedy_alg1.argtypes = [ctypes.c_int64, vp, vp, vp, ctypes.POINTER(ctypes.c_uint32)]
        lib.oracle_verify.argtypes = [ctypes.c_int64, vp, vp, vp, ctypes.POINTER(ctypes.c_int64)]
        lib.oracle_chromatic_bruteforce.argtypes = [ctypes.c_int64, vp, vp]
        for f in ("oracle_sgr", "oracle_greedy_alg1", "oracle_verify", "oracle_chromatic_bruteforce"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _csr(g):
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(g.col_idx, dtype=np.int32)
    if ci.size == 0:
        ci = np.zeros(1, dtype=np.int32)
    return rp, ci


def sgr(g, policy: str = "higher_id", max_rounds: int = 0, trace: bool = False):
    """Round-synchronous SGR (Alg. 7 / Alg. 2 with readings C1-C17).

    Returns (colors uint32[n], num_colors, rounds[, trace list of |W_r|]).
    """
    rp, ci = _csr(g)
    colors = np.zeros(max(g.n, 1), dtype=np.uint32)
    nc, rd = ctypes.c_uint32(), ctypes.c_uint32()
    cap = g.n + 2 if trace else 0
    tr = np.zeros(max(cap, 1), dtype=np.int64)
    rc = _load().oracle_sgr(g.n, rp.ctypes.data, ci.ctypes.data, POLICIES[policy], max_rounds,
                            colors.ctypes.data, ctypes.byref(nc), ctypes.byref(rd),
                            tr.ctypes.data if trace else None, cap)
    if rc == 3:
        raise NoConvergence(f"oracle_sgr: rounds exceeded max_rounds={max_rounds}")
    if rc != 0:
        raise RuntimeError(f"oracle_sgr failed: {rc}")
    out = (colors[:g.n], nc.value, rd.value)
    if trace:
        out = out + ([int(x) for x in tr[:rd.value]],)
    return out


def greedy_alg1(g):
    """Alg. 1 sequential greedy, ascending order."""
    rp, ci = _csr(g)
    colors = np.zeros(max(g.n, 1), dtype=np.uint32)
    nc = ctypes.c_uint32()
    rc = _load().oracle_greedy_alg1(g.n, rp.ctypes.data, ci.ctypes.data, colors.ctypes.data,
                                    ctypes.byref(nc))
    if rc != 0:
        raise RuntimeError(f"oracle_greedy_alg1 failed: {rc}")
    return colors[:g.n], nc.value


def verify(g, colors):
    """0 ok / 1 incomplete / 2 improper / 3 not First-Fit fixpoint; plus first bad vertex."""
    rp, ci = _csr(g)
    c = np.ascontiguousarray(colors, dtype=np.uint32)
    if c.size == 0:
        c = np.zeros(1, dtype=np.uint32)
    bad = ctypes.c_int64()
    rc = _load().oracle_verify(g.n, rp.ctypes.data, ci.ctypes.data, c.ctypes.data, ctypes.byref(bad))
    return rc, bad.value


def chromatic_bruteforce(g) -> int:
    rp, ci = _csr(g)
    return int(_load().oracle_chromatic_bruteforce(g.n, rp.ctypes.data, ci.ctypes.data))
