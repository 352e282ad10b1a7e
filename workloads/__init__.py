"""Seeded synthetic graph inputs shared by the CPU oracle and the CUDA path.

This module holds none of the coloring method's arithmetic: it only builds canonical
undirected CSR graphs (``row_ptr`` int64[n+1], ``col_idx`` int32[m]; SPEC.md:22-32,
PAPER.md:372-378 "CSR ... R and C").  The recipes (R-MAT PAPER.md:755-760, 27-point
stencil, 2-D mesh with edge deletion) are fixed in DESIGN.md "Input recipe".
Heavy generators live in ``gen.c`` (OpenMP, thread-count independent output).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import weakref
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libgcgen.so")
_SRC_GPU = os.path.join(_HERE, "gen_gpu.cu")
_LIB_GPU = os.path.join(_HERE, "libgcgen_gpu.so")
_lib = None
_lib_gpu = None


def build(force: bool = False, gpu: bool = True) -> str:
    """Compile gen.c into libgcgen.so (gcc -O3 -fopenmp) and gen_gpu.cu into libgcgen_gpu.so
    (nvcc, sm_100a)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    if gpu and (force or not os.path.exists(_LIB_GPU) or os.path.getmtime(_LIB_GPU) < os.path.getmtime(_SRC_GPU)):
        tmp = _LIB_GPU + f".tmp{os.getpid()}"
        nvcc = "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc"
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
                               "-shared", "-o", tmp, _SRC_GPU])
        os.replace(tmp, _LIB_GPU)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32pp = ctypes.POINTER(ctypes.POINTER(ctypes.c_int32))
        i64pp = ctypes.POINTER(ctypes.POINTER(ctypes.c_int64))
        lib.gen_rmat.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_uint64, i64p, i64p, i64pp, i32pp]
        lib.gen_rmat_range.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                       i64p, i64pp, i32pp]
        lib.gen_stencil27.argtypes = [ctypes.c_int32] * 3 + [i64p, i64p, i64pp, i32pp]
        lib.gen_mesh2d.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                   i64p, i64p, i64pp, i32pp]
        lib.gen_from_edges.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int64, i64p, i64pp, i32pp]
        lib.gen_rmat_perm.argtypes = [ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p]
        lib.gen_rmat_perm.restype = ctypes.c_int
        lib.gen_splitmix64.argtypes = [ctypes.c_uint64]
        lib.gen_splitmix64.restype = ctypes.c_uint64
        lib.gen_free.argtypes = [ctypes.c_void_p]
        for f in ("gen_rmat", "gen_rmat_range", "gen_stencil27", "gen_mesh2d", "gen_from_edges"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass
class Graph:
    """Canonical undirected CSR graph; ``m`` counts directed adjacency entries (C15)."""
    n: int
    row_ptr: np.ndarray  # int64 [n+1]
    col_idx: np.ndarray  # int32 [m]
    name: str = ""

    @property
    def m(self) -> int:
        return int(self.row_ptr[-1]) if self.n > 0 else 0

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def max_degree(self) -> int:
        return int(self.degrees().max()) if self.n > 0 else 0

    def adj(self, v: int) -> np.ndarray:
        return self.col_idx[self.row_ptr[v]:self.row_ptr[v + 1]]


def _adopt(ptr, count, dtype):
    """Wrap a malloc'd C array as a numpy array that frees it when collected."""
    if count == 0:
        _load().gen_free(ctypes.cast(ptr, ctypes.c_void_p))
        return np.zeros(0, dtype=dtype)
    arr = np.ctypeslib.as_array(ptr, shape=(count,))
    assert arr.dtype == dtype
    addr = ctypes.cast(ptr, ctypes.c_void_p).value
    weakref.finalize(arr, _load().gen_free, ctypes.c_void_p(addr))
    return arr


def _call(fn, *args):
    n = ctypes.c_int64()
    m = ctypes.c_int64()
    rp = ctypes.POINTER(ctypes.c_int64)()
    ci = ctypes.POINTER(ctypes.c_int32)()
    rc = fn(*args, ctypes.byref(n), ctypes.byref(m), ctypes.byref(rp), ctypes.byref(ci))
    if rc != 0:
        raise ValueError(f"generator failed with code {rc}")
    return n.value, _adopt(rp, n.value + 1, np.int64), _adopt(ci, m.value, np.int32)


def splitmix64(x: int) -> int:
    return int(_load().gen_splitmix64(ctypes.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


RMAT_G = (0.45, 0.15, 0.15)      # PAPER.md:760 rmat-g (d = 0.25)
RMAT_ER = (0.25, 0.25, 0.25)     # PAPER.md:759 rmat-er
GRAPH500 = (0.57, 0.19, 0.19)    # optional stress variant


def rmat(scale: int, edge_factor: int, abc=RMAT_G, seed: int = 1) -> Graph:
    a, b, c = abc
    n, rp, ci = _call(_load().gen_rmat, scale, edge_factor, a, b, c, seed)
    return Graph(n, rp, ci, f"rmat_s{scale}_ef{edge_factor}")


def rmat_range(scale: int, edge_factor: int, v_begin: int, v_end: int, abc=RMAT_G, seed: int = 1):
    """Rows [v_begin, v_end) of rmat(scale, edge_factor, abc, seed) without building the whole
    graph: (row_ptr int64[v_end-v_begin+1] rebased to 0, col_idx int32 in GLOBAL ids).  Used by
    the multi-GPU bench (each rank generates only its own vertex range) and for scale 27."""
    a, b, c = abc
    m = ctypes.c_int64()
    rp = ctypes.POINTER(ctypes.c_int64)()
    ci = ctypes.POINTER(ctypes.c_int32)()
    rc = _load().gen_rmat_range(scale, edge_factor, a, b, c, seed, v_begin, v_end, ctypes.byref(m),
                                ctypes.byref(rp), ctypes.byref(ci))
    if rc != 0:
        raise ValueError(f"gen_rmat_range failed with code {rc}")
    return _adopt(rp, v_end - v_begin + 1, np.int64), _adopt(ci, m.value, np.int32)


def rmat_perm(scale: int, seed: int = 1) -> np.ndarray:
    """The seeded Fisher-Yates relabelling of the W1 recipe (int32[2^scale])."""
    pi = np.empty(1 << scale, dtype=np.int32)
    rc = _load().gen_rmat_perm(scale, seed, pi.ctypes.data)
    if rc != 0:
        raise ValueError(f"gen_rmat_perm failed with code {rc}")
    return pi


def _load_gpu():
    global _lib_gpu
    if _lib_gpu is None:
        build()
        lib = ctypes.CDLL(_LIB_GPU)
        lib.gen_rmat_emit_gpu.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_ulonglong, ctypes.c_void_p, ctypes.c_longlong,
                                          ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong,
                                          ctypes.c_void_p]
        lib.gen_rmat_emit_gpu.restype = ctypes.c_int
        _lib_gpu = lib
    return _lib_gpu


def rmat_range_gpu(scale: int, edge_factor: int, v_begin: int, v_end: int, abc=RMAT_G, seed: int = 1,
                   device="cuda", chunk_arcs: int = 1 << 29):
    """Rows [v_begin, v_end) of rmat(scale, edge_factor, abc, seed), built on the GPU:
    (row_ptr int64[v_end-v_begin+1] rebased to 0, col_idx int32, global ids) as torch tensors on
    `device`.  Identical to rmat_range (tests/test_workloads.py).  Rows are produced in vertex
    chunks of at most about chunk_arcs arcs (each chunk: count pass, emit pass, sort, dedupe)."""
    import torch
    lib = _load_gpu()
    a, b, c = abc
    ab, abc_ = a + b, a + b + c
    n = 1 << scale
    ns = edge_factor * n
    dev = torch.device(device)
    pi = torch.from_numpy(rmat_perm(scale, seed)).to(dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)

    def arcs(cb, ce, keys=None):
        cnt.zero_()
        rc = lib.gen_rmat_emit_gpu(scale, ns, a, ab, abc_, seed, pi.data_ptr(), cb, ce, cnt.data_ptr(),
                                   keys.data_ptr() if keys is not None else None,
                                   keys.numel() if keys is not None else 0, stream)
        if rc != 0:
            raise RuntimeError(f"gen_rmat_emit_gpu: cudaError {rc}")
        return int(cnt.item())

    total = arcs(v_begin, v_end)
    nchunks = max(1, -(-total // chunk_arcs))
    cuts = [v_begin + (v_end - v_begin) * k // nchunks for k in range(nchunks + 1)]
    degs, cols = [], []
    for cb, ce in zip(cuts[:-1], cuts[1:]):
        k = arcs(cb, ce)
        keys = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
        assert arcs(cb, ce, keys) == k
        keys = torch.unique_consecutive(torch.sort(keys[:k]).values)
        degs.append(torch.bincount(keys >> 32, minlength=ce - cb) if k else torch.zeros(ce - cb, dtype=torch.int64,
                                                                                          device=dev))
        cols.append((keys & 0xFFFFFFFF).to(torch.int32) if k else torch.zeros(0, dtype=torch.int32, device=dev))
        del keys
    rp = torch.zeros(v_end - v_begin + 1, dtype=torch.int64, device=dev)
    if v_end > v_begin:
        torch.cumsum(torch.cat(degs), 0, out=rp[1:])
    ci = torch.cat(cols) if cols else torch.zeros(0, dtype=torch.int32, device=dev)
    return rp, ci


def stencil27(nx: int, ny: int | None = None, nz: int | None = None) -> Graph:
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    n, rp, ci = _call(_load().gen_stencil27, nx, ny, nz)
    return Graph(n, rp, ci, f"stencil27_{nx}x{ny}x{nz}")


def mesh2d(rows: int, cols: int, p_delete: float = 0.0, seed: int = 1) -> Graph:
    thr = 0 if p_delete <= 0 else int(p_delete * (1 << 64))
    thr = min(thr, (1 << 64) - 1)
    n, rp, ci = _call(_load().gen_mesh2d, rows, cols, thr, seed)
    return Graph(n, rp, ci, f"mesh_{rows}x{cols}_del{p_delete}")


def from_edges(n: int, edges, name: str = "") -> Graph:
    """Canonical CSR from an undirected edge list."""
    e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
    u = np.ascontiguousarray(e[:, 0])
    v = np.ascontiguousarray(e[:, 1])
    m = ctypes.c_int64()
    rp = ctypes.POINTER(ctypes.c_int64)()
    ci = ctypes.POINTER(ctypes.c_int32)()
    rc = _load().gen_from_edges(n, u.ctypes.data, v.ctypes.data, len(u), ctypes.byref(m),
                                ctypes.byref(rp), ctypes.byref(ci))
    if rc != 0:
        raise ValueError(f"from_edges failed with code {rc}")
    return Graph(n, _adopt(rp, n + 1, np.int64), _adopt(ci, m.value, np.int32), name)


# ---- small structured graphs (tests) -------------------------------------------------

def complete(n: int) -> Graph:
    return from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)], f"K{n}")


def path(n: int) -> Graph:
    return from_edges(n, [(i, i + 1) for i in range(n - 1)], f"P{n}")


def cycle(n: int) -> Graph:
    return from_edges(n, [(i, (i + 1) % n) for i in range(n)], f"C{n}")


def star(k: int, center_last: bool = False) -> Graph:
    c = k if center_last else 0
    leaves = range(k) if center_last else range(1, k + 1)
    return from_edges(k + 1, [(c, l) for l in leaves], f"star{k}{'_last' if center_last else ''}")


def edgeless(n: int) -> Graph:
    return Graph(n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), f"edgeless{n}")


def gnp(n: int, p: float, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < p
    return from_edges(n, np.stack([iu[keep], ju[keep]], 1), f"gnp{n}_{p}_{seed}")


def disjoint_union(*gs: Graph) -> Graph:
    edges, off = [], 0
    for g in gs:
        src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
        edges.append(np.stack([src + off, g.col_idx.astype(np.int64) + off], 1))
        off += g.n
    e = np.concatenate(edges) if edges else np.zeros((0, 2), np.int64)
    return from_edges(off, e, "union")


def relabel_reverse(g: Graph) -> Graph:
    """pi(v) = n-1-v (SURVEY.md §8(c) pin P12)."""
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
    e = np.stack([g.n - 1 - src, g.n - 1 - g.col_idx.astype(np.int64)], 1)
    return from_edges(g.n, e, g.name + "_rev")


def degree_stats(g: Graph):
    """Table 1 columns: n, m, min/max/avg degree, population variance."""
    d = g.degrees().astype(np.float64)
    return dict(n=g.n, m=g.m, min=int(d.min()), max=int(d.max()), avg=float(d.mean()),
                var=float(d.var()))


# ---- BASELINE.json configs ----------------------------------------------------------

CONFIGS = {
    # configs[0]: "R-MAT scale 16, edge factor 8 ... 1 GPU vs CPU oracle"
    "rmat16": lambda: rmat(16, 8),
    # configs[1]: "HPCG 27-point 3D stencil graph 128^3"
    "stencil128": lambda: stencil27(128),
    # configs[2]: "R-MAT scale 24, edge factor 16"
    "rmat24": lambda: rmat(24, 16),
    # configs[3]: "2D mesh with 30% random edge deletion, 8192x8192"
    "mesh8192": lambda: mesh2d(8192, 8192, 0.3),
    # configs[4]: "R-MAT scale 27, edge factor 16" (8 GPUs; not run in round 1)
    "rmat27": lambda: rmat(27, 16),
}


def config_graph(name: str) -> Graph:
    g = CONFIGS[name]()
    g.name = name
    return g
