"""B200-native round-synchronous speculative-greedy (SGR) graph colouring (arXiv 1606.06025).

Thin Python binding over the C ABI in ``include/gc.h`` (``csrc/libgc.so``): argument
marshalling only — every step of the colouring runs in the library's sm_100a kernels.
There is no CPU fallback: importing this module raises if the CUDA library is missing,
and the calls fail loudly without a GPU.

    import paper_1606_06025_b200 as gc
    res = gc.color(row_ptr, col_idx)          # torch CUDA tensors (int64 / int32)
    res.colors, res.num_colors, res.rounds
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

from ._build import LIB_PATH, build, load  # noqa: F401

_lib = load()

POLICIES = {"higher_id": 0, "lower_id": 1, "degree": 2}
FLAG_VALIDATE = 1
FLAG_VALIDATE_SYMMETRY = 2
FLAG_TRACE = 4
FLAG_PULL_FIRSTFIT = 8
FLAG_HOST_ROUNDS = 16
FLAG_COUNT_WORK = 32

STATUS = {0: "GC_OK", 1: "GC_ERR_INVALID_ARGUMENT", 2: "GC_ERR_INVALID_GRAPH",
          3: "GC_ERR_NO_CONVERGENCE", 4: "GC_ERR_OUT_OF_MEMORY", 5: "GC_ERR_CUDA",
          6: "GC_ERR_NCCL", 7: "GC_ERR_UNSUPPORTED"}


class GcError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


class Work(ctypes.Structure):
    _fields_ = [("phase_a_vertices", ctypes.c_uint64), ("phase_a_edges", ctypes.c_uint64),
                ("phase_b_vertices", ctypes.c_uint64), ("phase_b_edges", ctypes.c_uint64),
                ("phase_b_gathers", ctypes.c_uint64), ("commit_scatter", ctypes.c_uint64),
                ("pushes", ctypes.c_uint64), ("scatter_reds", ctypes.c_uint64),
                ("dense_a_swept", ctypes.c_uint64), ("dense_b_swept", ctypes.c_uint64),
                ("sparse_a_entries", ctypes.c_uint64), ("sparse_b_entries", ctypes.c_uint64),
                ("state_bytes", ctypes.c_uint64), ("phase_b_evaluated", ctypes.c_uint64),
                ("dense_b_evaluated", ctypes.c_uint64), ("dirty_marks", ctypes.c_uint64),
                ("tent_changes", ctypes.c_uint64), ("pending_degree_sum", ctypes.c_uint64),
                ("reserved", ctypes.c_uint64 * 3)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_ if k != "reserved"}


class Tuning(ctypes.Structure):
    """gc_tuning (include/gc.h): schedule overrides; -1 = measured default."""
    _fields_ = [("struct_size", ctypes.c_uint32), ("state_bytes", ctypes.c_int32),
                ("dense_div", ctypes.c_int32), ("dense_div_n1", ctypes.c_int32), ("n1", ctypes.c_int32),
                ("list", ctypes.c_int32), ("compact", ctypes.c_int32), ("scatter_filter", ctypes.c_int32),
                ("dch", ctypes.c_int32), ("n1_chg", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("watchdog_ms", ctypes.c_int32), ("widen", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


class Opts(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("policy", ctypes.c_uint32),
                ("flags", ctypes.c_uint32), ("max_rounds", ctypes.c_uint32),
                ("device", ctypes.c_int32), ("thread_bin_max", ctypes.c_uint32),
                ("warp_bin_max", ctypes.c_uint32), ("blocks_per_sm", ctypes.c_uint32),
                ("stream", ctypes.c_void_p), ("trace_worklist", ctypes.c_void_p),
                ("trace_capacity", ctypes.c_uint32), ("group_bin_max", ctypes.c_uint32),
                ("work", ctypes.POINTER(Work)), ("kernel_ms", ctypes.POINTER(ctypes.c_float)),
                ("phase_ns", ctypes.c_void_p), ("tuning", ctypes.POINTER(Tuning)),
                ("reserved", ctypes.c_uint64 * 1)]


_vp = ctypes.c_void_p
_lib.gc_opts_default.argtypes = [ctypes.POINTER(Opts)]
_lib.gc_opts_default.restype = None
_lib.gc_tuning_default.argtypes = [ctypes.POINTER(Tuning)]
_lib.gc_tuning_default.restype = None
_lib.gc_color.argtypes = [ctypes.c_int64, _vp, _vp, ctypes.POINTER(Opts), _vp,
                          ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
_lib.gc_color.restype = ctypes.c_int
_lib.gc_verify.argtypes = [ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]
_lib.gc_verify.restype = ctypes.c_int
_lib.gc_status_string.argtypes = [ctypes.c_int]
_lib.gc_status_string.restype = ctypes.c_char_p
_lib.gc_last_error_message.argtypes = []
_lib.gc_last_error_message.restype = ctypes.c_char_p
_lib.gc_partition_edge_balanced.argtypes = [ctypes.c_int64, _vp, ctypes.c_int32, _vp]
_lib.gc_partition_edge_balanced.restype = ctypes.c_int
_lib.gc_abi_version.argtypes = []
_lib.gc_abi_version.restype = ctypes.c_int32

assert ctypes.sizeof(Opts) == 96, ctypes.sizeof(Opts)
assert ctypes.sizeof(Tuning) == 64, ctypes.sizeof(Tuning)


def _err(status: int):
    raise GcError(status, _lib.gc_last_error_message().decode(errors="replace"))


def _ptr(a):
    """Data pointer of a torch tensor or numpy array (argument marshalling only)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _is_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and a.is_cuda


@dataclass
class ColorResult:
    colors: object            # uint32 colours: torch.int32 CUDA tensor (bit view) or numpy uint32
    num_colors: int
    rounds: int
    trace: list | None = None
    work: dict | None = field(default=None)
    kernel_ms: float | None = None
    phase_us: list | None = None     # per round (Phase A us, Phase B us) with phase_times=True


def default_opts() -> Opts:
    o = Opts()
    _lib.gc_opts_default(ctypes.byref(o))
    return o


def make_tuning(tuning: dict | None):
    """gc_tuning from a dict of its field names (None -> NULL: the measured defaults)."""
    if not tuning:
        return None
    t = Tuning()
    _lib.gc_tuning_default(ctypes.byref(t))
    for k, v in tuning.items():
        if k not in dict(Tuning._fields_) or k in ("struct_size", "reserved"):
            raise ValueError(f"unknown gc_tuning field {k!r}")
        setattr(t, k, int(v))
    return t


def color(row_ptr, col_idx, policy: str = "higher_id", validate: bool = True,
          symmetry: bool = False, pull_firstfit: bool = False, host_rounds: bool = False,
          trace: bool = False, count_work: bool = False, max_rounds: int = 0,
          thread_bin_max: int = 0, group_bin_max: int = 0, warp_bin_max: int = 0, blocks_per_sm: int = 0,
          stream=None, device: int | None = None, out=None, time_kernel: bool = False,
          phase_times: bool = False, tuning: dict | None = None) -> ColorResult:
    """gc_color(n, row_ptr, col_idx, opts, colors_out, &num_colors, &rounds) (include/gc.h).

    row_ptr: int64[n+1], col_idx: int32[m] — torch tensors (CUDA or CPU) or numpy arrays.
    Device inputs give a CUDA int32 tensor holding the uint32 colours; host inputs give a
    numpy uint32 array (the library copies host inputs in and the colours back).
    """
    import numpy as np
    n = int(row_ptr.shape[0]) - 1
    trace = trace or phase_times
    o = default_opts()
    o.policy = POLICIES[policy]
    o.flags = ((FLAG_VALIDATE if validate else 0) | (FLAG_VALIDATE_SYMMETRY if symmetry else 0)
               | (FLAG_PULL_FIRSTFIT if pull_firstfit else 0) | (FLAG_HOST_ROUNDS if host_rounds else 0)
               | (FLAG_TRACE if trace else 0) | (FLAG_COUNT_WORK if count_work else 0))
    o.max_rounds = max_rounds
    o.thread_bin_max = thread_bin_max
    o.warp_bin_max = warp_bin_max
    o.group_bin_max = group_bin_max
    o.blocks_per_sm = blocks_per_sm
    tun = make_tuning(tuning)
    if tun is not None:
        o.tuning = ctypes.pointer(tun)
    dev_inputs = _is_cuda(row_ptr)
    if dev_inputs:
        import torch
        dev_index = row_ptr.device.index if device is None else device
        o.device = dev_index
        if stream is None:
            stream = torch.cuda.current_stream(row_ptr.device).cuda_stream
        if out is None:
            out = torch.empty(max(n, 1), dtype=torch.int32, device=row_ptr.device)
    else:
        o.device = -1 if device is None else device
        if out is None:
            out = np.zeros(max(n, 1), dtype=np.uint32)
    o.stream = stream
    tr = None
    ph = None
    if phase_times:
        ph = np.zeros(4 * max(n + 2, 1) + 1, dtype=np.uint64)
        o.phase_ns = ph.ctypes.data
    if trace:
        tr = np.zeros(max(n + 2, 1), dtype=np.uint32)
        o.trace_worklist = tr.ctypes.data
        o.trace_capacity = len(tr)
    wk = Work()
    if count_work:
        o.work = ctypes.pointer(wk)
    kms = ctypes.c_float(0)
    if time_kernel:
        o.kernel_ms = ctypes.pointer(kms)
    nc, rd = ctypes.c_uint32(), ctypes.c_uint32()
    st = _lib.gc_color(n, _ptr(row_ptr), _ptr(col_idx), ctypes.byref(o), _ptr(out),
                       ctypes.byref(nc), ctypes.byref(rd))
    if st != 0:
        _err(st)
    res = ColorResult(out[:n], nc.value, rd.value)
    if trace:
        res.trace = [int(x) for x in tr[:rd.value]]
    if count_work:
        res.work = wk.as_dict()
    if time_kernel:
        res.kernel_ms = float(kms.value)
    if phase_times:
        # per round: (Phase A us, Phase B us) barrier to barrier, and the part of each spent
        # after the last CTA finished its work (barrier + tail): (A, B, A_wait, B_wait)
        t = ph[:4 * rd.value + 1].astype(np.int64)
        out = []
        for r in range(1, rd.value + 1):
            a0 = t[4 * r - 4]  # previous barrier (or ingest end)
            a = (t[4 * r - 2] - a0) / 1e3 if r > 1 else 0.0
            aw = (t[4 * r - 2] - t[4 * r - 3]) / 1e3 if r > 1 else 0.0
            bstart = t[4 * r - 2] if r > 1 else t[0]
            out.append((a, (t[4 * r] - bstart) / 1e3, aw, (t[4 * r] - t[4 * r - 1]) / 1e3))
        res.phase_us = out
    return res


def verify(row_ptr, col_idx, colors, device: int = -1) -> int:
    """gc_verify: -1 when colors is complete, proper and a First-Fit fixpoint, else a bad vertex."""
    n = int(row_ptr.shape[0]) - 1
    bad = ctypes.c_int64()
    st = _lib.gc_verify(n, _ptr(row_ptr), _ptr(col_idx), _ptr(colors), device, ctypes.byref(bad))
    if st not in (0, 2):
        _err(st)
    return int(bad.value)


def partition_edge_balanced(row_ptr, parts: int):
    """gc_partition_edge_balanced on a host int64 row_ptr -> numpy int64 bounds[parts+1]."""
    import numpy as np
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    bounds = np.zeros(parts + 1, dtype=np.int64)
    st = _lib.gc_partition_edge_balanced(len(rp) - 1, rp.ctypes.data, parts, bounds.ctypes.data)
    if st != 0:
        _err(st)
    return bounds


_lib.gc__bench_grid_sync.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_float)]
_lib.gc__bench_grid_sync.restype = ctypes.c_int


def bench_grid_sync(device: int = 0, blocks_per_sm: int = 0, iters: int = 2000) -> float:
    """Diagnostics: microseconds per grid barrier of the persistent kernel."""
    us = ctypes.c_float()
    st = _lib.gc__bench_grid_sync(device, blocks_per_sm, iters, ctypes.byref(us))
    if st != 0:
        _err(st)
    return float(us.value)


def status_string(s: int) -> str:
    return _lib.gc_status_string(s).decode()


def abi_version() -> int:
    return int(_lib.gc_abi_version())
