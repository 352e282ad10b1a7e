"""C-ABI library: builds for sm_100a, loads, exports every symbol include/gc.h declares;
host-only logic (argument checks, edge-balanced partition) — no GPU needed."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import workloads as wl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = "".join(open(os.path.join(ROOT, "include", h)).read() for h in ("gc.h", "gc_dist.h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_call():
    syms = _declared_symbols()
    for s in ("gc_color", "gc_verify", "gc_opts_default", "gc_status_string",
              "gc_last_error_message", "gc_partition_edge_balanced", "gc_abi_version",
              "gc_tuning_default", "gc_comm_init", "gc_color_dist", "gc_comm_destroy",
              "gc_comm_init_local", "gc_nccl_unique_id"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1606_06025_b200 as gc
    out = subprocess.check_output(["nm", "-D", "--defined-only", gc.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (gc_\w+)", out))
    missing = [s for s in _declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_is_sm100a():
    import paper_1606_06025_b200 as gc
    out = subprocess.check_output(["cuobjdump", "--list-elf", gc.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_opts_layout_and_defaults():
    import paper_1606_06025_b200 as gc
    o = gc.default_opts()
    assert o.struct_size == ctypes.sizeof(gc.Opts) == 96
    assert o.policy == 0 and o.flags == gc.FLAG_VALIDATE and o.device == -1
    assert gc.abi_version() == 2
    t = gc.make_tuning(dict(n1=2))
    assert t.struct_size == 64 and t.n1 == 2 and t.dense_div == -1 and t.variant == -1
    with pytest.raises(ValueError):
        gc.make_tuning(dict(bogus=1))
    assert gc.status_string(2) == "GC_ERR_INVALID_GRAPH"


def test_invalid_arguments_rejected_before_any_cuda_call():
    import paper_1606_06025_b200 as gc
    lib = gc._lib
    nc, rd = ctypes.c_uint32(7), ctypes.c_uint32(7)
    assert lib.gc_color(-1, None, None, None, None, ctypes.byref(nc), ctypes.byref(rd)) == 1
    assert nc.value == 0 and rd.value == 0
    assert lib.gc_color(5, None, None, None, None, ctypes.byref(nc), ctypes.byref(rd)) == 1
    assert b"NULL" in lib.gc_last_error_message()
    assert lib.gc_color(1 << 31, None, None, None, None, ctypes.byref(nc), ctypes.byref(rd)) == 1
    o = gc.default_opts()
    o.struct_size = 12
    assert lib.gc_color(3, None, None, ctypes.byref(o), None, ctypes.byref(nc), ctypes.byref(rd)) == 1
    o = gc.default_opts()
    o.policy = 9
    assert lib.gc_color(3, None, None, ctypes.byref(o), None, ctypes.byref(nc), ctypes.byref(rd)) == 1
    # n = 0 is a valid empty graph
    assert lib.gc_color(0, None, None, None, None, ctypes.byref(nc), ctypes.byref(rd)) == 0
    assert lib.gc_color(3, None, None, None, None, None, None) == 1


def test_partition_edge_balanced():
    import paper_1606_06025_b200 as gc
    g = wl.rmat(12, 8)
    m = g.m
    for parts in (1, 2, 3, 4, 8, 16):
        b = gc.partition_edge_balanced(g.row_ptr, parts)
        assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b) >= 0)
        for k in range(1, parts):
            target = -(-k * m // parts)
            v = b[k]
            assert g.row_ptr[v] >= target and (v == 0 or g.row_ptr[v - 1] < target)
    b = gc.partition_edge_balanced(np.zeros(1, np.int64), 4)
    assert b.tolist() == [0, 0, 0, 0, 0]
    with pytest.raises(gc.GcError):
        gc.partition_edge_balanced(g.row_ptr, 0)
