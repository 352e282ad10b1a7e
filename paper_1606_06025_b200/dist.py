"""Multi-GPU (vertex-range partitioned) SGR colouring — round driver over include/gc_dist.h.

One partition per process/GPU (torchrun; NCCL over NVLink for the two per-round
all-gathers), or several partitions inside one process (used by the partition-invariance
tests on one GPU).  SURVEY §8(e): edge-balanced contiguous vertex ranges, replicated (ghost)
state words, two exchanges per round, global ids decide conflicts; the colouring equals the
single-GPU one for any cover of [0, n).

The round loop here is host orchestration only; every per-vertex step runs in the library's
kernels (gc_dist_phase_a / _phase_b / _pack / _unpack).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib, _err, _ptr, default_opts, POLICIES, partition_edge_balanced

_vp = ctypes.c_void_p
_lib.gc_dist_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp]
_lib.gc_dist_phase_a.argtypes = [_vp]
_lib.gc_dist_phase_b.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint32)]
_lib.gc_dist_pack.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.POINTER(ctypes.c_uint64)]
_lib.gc_dist_unpack.argtypes = [_vp, _vp, ctypes.c_uint64]
_lib.gc_dist_next_round.argtypes = [_vp]
_lib.gc_dist_finalize.argtypes = [_vp, _vp, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
_lib.gc_dist_destroy.argtypes = [_vp]
for _f in ("gc_dist_create", "gc_dist_phase_a", "gc_dist_phase_b", "gc_dist_pack", "gc_dist_unpack",
           "gc_dist_next_round", "gc_dist_finalize", "gc_dist_destroy"):
    getattr(_lib, _f).restype = ctypes.c_int


def local_slice(row_ptr, col_idx, v_begin: int, v_end: int):
    """Rows [v_begin, v_end) of a CSR: (row_ptr rebased to 0, col_idx in global ids).
    Works on numpy arrays or torch tensors (slicing / subtraction only)."""
    b, e = int(row_ptr[v_begin]), int(row_ptr[v_end])
    return row_ptr[v_begin:v_end + 1] - b, col_idx[b:e]


class CudaPartition:
    """One partition's state on one GPU (wraps a gc_dist handle)."""

    def __init__(self, n_global: int, v_begin: int, v_end: int, row_ptr_local, col_idx_local,
                 policy: str = "higher_id", device: int | None = None):
        import torch
        self.n_global, self.v_begin, self.v_end = n_global, v_begin, v_end
        self.dev = row_ptr_local.device
        self._keep = (row_ptr_local, col_idx_local)
        o = default_opts()
        o.policy = POLICIES[policy]
        o.device = self.dev.index if device is None else device
        h = _vp()
        st = _lib.gc_dist_create(ctypes.byref(h), n_global, v_begin, v_end, _ptr(row_ptr_local),
                                 _ptr(col_idx_local), ctypes.byref(o))
        if st != 0:
            _err(st)
        self.h = h
        nl = max(v_end - v_begin, 1)
        self.pairs = torch.empty(2 * nl, dtype=torch.int32, device=self.dev)

    def phase_a(self):
        st = _lib.gc_dist_phase_a(self.h)
        if st != 0:
            _err(st)

    def phase_b(self) -> int:
        c = ctypes.c_uint32()
        st = _lib.gc_dist_phase_b(self.h, ctypes.byref(c))
        if st != 0:
            _err(st)
        return int(c.value)

    def pack(self, what: int):
        c = ctypes.c_uint64()
        st = _lib.gc_dist_pack(self.h, what, _ptr(self.pairs), ctypes.byref(c))
        if st != 0:
            _err(st)
        return self.pairs[:2 * c.value]

    def unpack(self, pairs):
        pairs = pairs.to(self.dev).contiguous()
        st = _lib.gc_dist_unpack(self.h, _ptr(pairs) if pairs.numel() else None, pairs.numel() // 2)
        if st != 0:
            _err(st)

    def next_round(self):
        st = _lib.gc_dist_next_round(self.h)
        if st != 0:
            _err(st)

    def finalize(self):
        import torch
        out = torch.empty(max(self.v_end - self.v_begin, 1), dtype=torch.int32, device=self.dev)
        mx, rd = ctypes.c_uint32(), ctypes.c_uint32()
        st = _lib.gc_dist_finalize(self.h, _ptr(out), ctypes.byref(mx), ctypes.byref(rd))
        if st != 0:
            _err(st)
        return out[:self.v_end - self.v_begin], int(mx.value), int(rd.value)

    def close(self):
        if getattr(self, "h", None):
            _lib.gc_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalComm:
    """All partitions live in this process (world of one process)."""

    def allgather(self, t):
        return t

    def allreduce_sum(self, x: int) -> int:
        return int(x)

    def allreduce_max(self, x: int) -> int:
        return int(x)


class TorchComm:
    """torch.distributed process group (NCCL on GPUs, gloo on CPU) — plumbing only."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)

    def allgather(self, t):
        import torch
        dist = self.dist
        k = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        sizes = [torch.zeros_like(k) for _ in range(self.world)]
        dist.all_gather(sizes, k, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        mx = max(sizes) if sizes else 0
        if mx == 0:
            return t[:0]
        buf = torch.zeros(mx, dtype=t.dtype, device=t.device)
        buf[:t.numel()] = t
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return torch.cat([o[:s] for o, s in zip(outs, sizes)])

    def _reduce(self, x: int, op) -> int:
        import torch
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(x)], dtype=torch.int64, device=dev)
        self.dist.all_reduce(t, op=op, group=self.group)
        return int(t.item())

    def allreduce_sum(self, x: int) -> int:
        return self._reduce(x, self.dist.ReduceOp.SUM)

    def allreduce_max(self, x: int) -> int:
        return self._reduce(x, self.dist.ReduceOp.MAX)


@dataclass
class DistResult:
    colors_local: list          # per local partition: colours of its rows
    num_colors: int
    rounds: int
    exchanged_pairs: int        # (vertex, word) pairs this process contributed


def _exchange(parts, comm, what: int) -> int:
    import torch
    packed = [p.pack(what) for p in parts]
    local = torch.cat(packed) if len(packed) > 1 else packed[0]
    everything = comm.allgather(local)
    for p in parts:
        p.unpack(everything)
    return local.numel() // 2


def run_rounds(parts, comm) -> DistResult:
    """The SGR round loop over this process's partitions (SURVEY §8(e) per-round steps)."""
    r = 1
    sent = 0
    while True:
        if r > 1:
            for p in parts:
                p.phase_a()
            sent += _exchange(parts, comm, 0)          # exchange #1: tentative colours
        local_next = sum(p.phase_b() for p in parts)
        sent += _exchange(parts, comm, 1)              # exchange #2: commits
        if comm.allreduce_sum(local_next) == 0:
            break
        for p in parts:
            p.next_round()
        r += 1
    outs = [p.finalize() for p in parts]
    mx = comm.allreduce_max(max(o[1] for o in outs))
    rounds = outs[0][2]
    return DistResult([o[0] for o in outs], mx, rounds, sent)


def color_partitioned(row_ptr, col_idx, parts: int, policy: str = "higher_id"):
    """Colour one graph as `parts` edge-balanced partitions inside this process (one GPU).
    Used to check partition invariance; returns (colours, num_colors, rounds)."""
    import numpy as np
    import torch
    n = int(row_ptr.shape[0]) - 1
    rp_host = row_ptr.cpu().numpy() if hasattr(row_ptr, "cpu") else np.asarray(row_ptr)
    bounds = partition_edge_balanced(rp_host, parts)
    objs = []
    for k in range(parts):
        b, e = int(bounds[k]), int(bounds[k + 1])
        rpl, cil = local_slice(row_ptr, col_idx, b, e)
        objs.append(CudaPartition(n, b, e, rpl.contiguous(), cil.contiguous(), policy))
    res = run_rounds(objs, LocalComm())
    colors = torch.cat(res.colors_local) if res.colors_local else torch.zeros(0, dtype=torch.int32)
    for o in objs:
        o.close()
    return colors, res.num_colors, res.rounds
