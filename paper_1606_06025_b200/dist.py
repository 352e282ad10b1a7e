"""Multi-GPU SGR colouring — binding of include/gc_dist.h (SURVEY §8(b) multi-GPU calls).

One rank per GPU (torchrun); the library runs the whole colouring as one persistent kernel per
rank with a device-initiated exchange over NVLink peer memory and uses NCCL
only to bootstrap.  torch.distributed is used for exactly one thing here: broadcasting the
NCCL unique id (``init_from_torch``).  Edge-balanced contiguous vertex ranges
(``partition_edge_balanced``); any cover gives colours bit-identical to one GPU.

``local_group`` emulates ``world`` ranks inside one process on one GPU (each rank's
``color_dist`` runs on its own host thread): the same kernels, windows, peer stores and
cross-rank barriers — used by the partition-invariance tests on the single-GPU test box.

Everything here is argument marshalling and host bookkeeping (ranges, slices, assembling the
gathered colours); every per-vertex step runs in the library's kernels.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import (FLAG_COUNT_WORK, FLAG_TRACE, FLAG_VALIDATE, POLICIES, ColorResult, Work, _err, _is_cuda, _lib,
               _ptr, default_opts, make_tuning, partition_edge_balanced)

_vp = ctypes.c_void_p
MAX_RANKS = 8
UNIQUE_ID_BYTES = 128

_lib.gc_nccl_unique_id.argtypes = [_vp]
_lib.gc_comm_init.argtypes = [ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32]
_lib.gc_comm_init_local.argtypes = [ctypes.POINTER(_vp), ctypes.c_int32, ctypes.c_int32]
_lib.gc_color_dist.argtypes = [_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp, _vp,
                               ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
_lib.gc_comm_destroy.argtypes = [_vp]
for _f in ("gc_nccl_unique_id", "gc_comm_init", "gc_comm_init_local", "gc_color_dist", "gc_comm_destroy"):
    getattr(_lib, _f).restype = ctypes.c_int

__all__ = ["Comm", "nccl_unique_id", "init_from_torch", "local_group", "color_dist", "local_slice",
           "color_partitioned_local", "assemble", "partition_edge_balanced"]


class Comm:
    """A gc_comm handle (one rank)."""

    def __init__(self, handle, rank: int, world: int, device: int):
        self.h, self.rank, self.world, self.device = handle, rank, world, device

    def close(self):
        if self.h:
            _lib.gc_comm_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(UNIQUE_ID_BYTES)
    st = _lib.gc_nccl_unique_id(buf)
    if st != 0:
        _err(st)
    return buf.raw


def comm_init(rank: int, world: int, uid: bytes, device: int) -> Comm:
    """gc_comm_init (collective over the world's processes)."""
    if len(uid) != UNIQUE_ID_BYTES:
        raise ValueError("uid must be the 128 bytes of gc_nccl_unique_id")
    h = _vp()
    st = _lib.gc_comm_init(ctypes.byref(h), rank, world, ctypes.create_string_buffer(uid, UNIQUE_ID_BYTES), device)
    if st != 0:
        _err(st)
    return Comm(h, rank, world, device)


def broadcast_uid(make_uid, group=None) -> bytes:
    """Rank 0 creates the id, every rank returns it (torch.distributed object broadcast; any
    backend).  Host logic only — tested with gloo on CPU."""
    import torch.distributed as dist
    obj = [make_uid() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_from_torch(device: int | None = None, group=None) -> Comm:
    """gc_comm_init for this process of an initialised torch.distributed world."""
    import torch
    import torch.distributed as dist
    dev = torch.cuda.current_device() if device is None else device
    uid = broadcast_uid(nccl_unique_id, group)
    return comm_init(dist.get_rank(group), dist.get_world_size(group), uid, dev)


def local_group(world: int, device: int = 0) -> list:
    """gc_comm_init_local: `world` emulated ranks on one GPU, one process."""
    hs = (_vp * world)()
    st = _lib.gc_comm_init_local(hs, world, device)
    if st != 0:
        _err(st)
    return [Comm(_vp(hs[q]), q, world, device) for q in range(world)]


def local_slice(row_ptr, col_idx, v_begin: int, v_end: int):
    """Rows [v_begin, v_end) of a CSR: (row_ptr rebased to 0, col_idx in global ids).
    Works on numpy arrays or torch tensors (slicing / subtraction only)."""
    b, e = int(row_ptr[v_begin]), int(row_ptr[v_end])
    return row_ptr[v_begin:v_end + 1] - b, col_idx[b:e]


def color_dist(comm: Comm, n_global: int, v_begin: int, v_end: int, row_ptr_local, col_idx_local,
               policy: str = "higher_id", validate: bool = True, trace: bool = False,
               count_work: bool = False, max_rounds: int = 0, out=None, stream=None,
               time_kernel: bool = False, tuning: dict | None = None) -> ColorResult:
    """gc_color_dist: colours of this rank's rows (colors = local range); num_colors, rounds
    (and the |W_r| trace) are global and identical on every rank.  Collective."""
    nl = v_end - v_begin
    o = default_opts()
    o.policy = POLICIES[policy]
    o.flags = ((FLAG_VALIDATE if validate else 0) | (FLAG_TRACE if trace else 0)
               | (FLAG_COUNT_WORK if count_work else 0))
    o.max_rounds = max_rounds
    o.device = comm.device
    tun = make_tuning(tuning)
    if tun is not None:
        o.tuning = ctypes.pointer(tun)
    if out is None:
        if _is_cuda(row_ptr_local):
            import torch
            out = torch.empty(max(nl, 1), dtype=torch.int32, device=row_ptr_local.device)
        else:
            out = np.zeros(max(nl, 1), dtype=np.uint32)
    if stream is not None:
        o.stream = stream
    tr = None
    if trace:
        tr = np.zeros(max(n_global + 2, 1), dtype=np.uint32)
        o.trace_worklist = tr.ctypes.data
        o.trace_capacity = len(tr)
    wk = Work()
    if count_work:
        o.work = ctypes.pointer(wk)
    kms = ctypes.c_float(0)
    if time_kernel:
        o.kernel_ms = ctypes.pointer(kms)
    nc, rd = ctypes.c_uint32(), ctypes.c_uint32()
    st = _lib.gc_color_dist(comm.h, n_global, v_begin, v_end, _ptr(row_ptr_local), _ptr(col_idx_local),
                            ctypes.byref(o), _ptr(out), ctypes.byref(nc), ctypes.byref(rd))
    if st != 0:
        _err(st)
    res = ColorResult(out[:nl], nc.value, rd.value)
    if trace:
        res.trace = [int(x) for x in tr[:rd.value]]
    if count_work:
        res.work = wk.as_dict()
    if time_kernel:
        res.kernel_ms = float(kms.value)
    return res


def assemble(parts, bounds):
    """Concatenate per-rank colour arrays (rank order) into the global array, checking that
    they tile [0, n) as bounds says (host logic)."""
    assert len(parts) == len(bounds) - 1
    for q, c in enumerate(parts):
        assert len(c) == int(bounds[q + 1]) - int(bounds[q]), (q, len(c))
    return np.concatenate([np.asarray(c, dtype=np.uint32) for c in parts]) if parts else np.zeros(0, np.uint32)


def color_partitioned_local(row_ptr, col_idx, bounds, policy: str = "higher_id", device: int = 0, comms=None,
                            **kw):
    """Colour a device-resident graph as len(bounds)-1 emulated ranks on one GPU (local group,
    one host thread per rank; ctypes releases the GIL during the call).  Returns (global
    colours as numpy uint32, per-rank ColorResults)."""
    world = len(bounds) - 1
    own = comms is None
    comms = local_group(world, device) if own else comms
    n = int(row_ptr.shape[0]) - 1
    results, errors = [None] * world, [None] * world
    slices = []
    for q in range(world):  # the inputs are made before the ranks start (as separate processes would)
        b, e = int(bounds[q]), int(bounds[q + 1])
        rpl, cil = local_slice(row_ptr, col_idx, b, e)
        if _is_cuda(rpl):
            rpl = rpl.contiguous()
            cil = cil.contiguous() if cil.numel() else cil.new_zeros(1)
        slices.append((b, e, rpl, cil))

    def run(q):
        b, e, rpl, cil = slices[q]
        try:
            results[q] = color_dist(comms[q], n, b, e, rpl, cil, policy=policy, **kw)
        except Exception as ex:  # collected and re-raised on the caller's thread
            errors[q] = ex

    th = [threading.Thread(target=run, args=(q,)) for q in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if own:
        for c in comms:
            c.close()
    bad = [(q, ex) for q, ex in enumerate(errors) if ex is not None]
    if bad:
        q0, ex0 = bad[0]
        if len(bad) > 1:  # every rank's error (the first is often a consequence of another's)
            ex0.args = (ex0.args[0] + " | " + " | ".join(f"rank {q}: {ex}" for q, ex in bad[1:]),)
        raise ex0
    parts = []
    for r in results:
        c = r.colors
        parts.append(c.cpu().numpy().view(np.uint32) if hasattr(c, "cpu") else np.asarray(c, np.uint32))
    return assemble(parts, bounds), results
