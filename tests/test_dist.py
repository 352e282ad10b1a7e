"""Multi-GPU path: include/gc_dist.h (gc_comm_init / gc_color_dist / gc_comm_destroy) and its
binding paper_1606_06025_b200/dist.py.

CPU (no GPU; gloo world_size 2 where processes are involved): the host logic around the
library — NCCL unique-id broadcast over torch.distributed, edge-balanced bounds, local CSR
slices in global ids, assembling the ranks' colour ranges — and the library's argument checks
that run before any CUDA call.  The gloo test colours each rank's range with the CPU oracle
restricted to that range (test infrastructure), so the gathered result must equal the oracle.

GPU: the real device-initiated kernels on the single test GPU through the
one-process emulation (gc_comm_init_local: `world` ranks, one host thread each, every rank's
persistent kernel resident side by side, peer stores into sibling windows, cross-rank
barriers): colours, num_colors, rounds and |W_r| trace must equal the oracle's for every
cover of [0, n) — edge-balanced, random, with empty ranges — every policy and every schedule
knob (partition invariance).
"""
import ctypes
import os
import socket

import numpy as np
import pytest

import oracle
import workloads as wl

POLICIES = ["higher_id", "lower_id", "degree"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def random_bounds(n, parts, seed):
    """A cover of [0, n) by `parts` contiguous ranges (some possibly empty)."""
    rng = np.random.default_rng(seed)
    cuts = np.sort(rng.integers(0, n + 1, parts - 1))
    return np.concatenate([[0], cuts, [n]]).astype(np.int64)


# ---------------------------------------------------------------- CPU: host logic

def test_local_slice_and_assemble():
    from paper_1606_06025_b200 import partition_edge_balanced
    from paper_1606_06025_b200.dist import assemble, local_slice
    g = wl.rmat(9, 8)
    for bounds in (partition_edge_balanced(g.row_ptr, 3), random_bounds(g.n, 5, 1),
                   np.array([0, 0, g.n, g.n], np.int64)):
        rebuilt, parts = [], []
        for k in range(len(bounds) - 1):
            b, e = int(bounds[k]), int(bounds[k + 1])
            rpl, cil = local_slice(g.row_ptr, g.col_idx, b, e)
            assert rpl[0] == 0 and rpl[-1] == len(cil)
            rebuilt.append(cil)
            parts.append(np.arange(b, e, dtype=np.uint32))
        assert np.array_equal(np.concatenate(rebuilt), g.col_idx)
        assert np.array_equal(assemble(parts, bounds), np.arange(g.n, dtype=np.uint32))


def test_dist_argument_checks_without_gpu():
    import paper_1606_06025_b200 as gc
    import paper_1606_06025_b200.dist  # noqa: F401  (declares the argtypes)
    lib = gc._lib
    nc, rd = ctypes.c_uint32(5), ctypes.c_uint32(5)
    assert lib.gc_color_dist(None, 10, 0, 10, None, None, None, None, ctypes.byref(nc), ctypes.byref(rd)) == 1
    hs = (ctypes.c_void_p * 9)()
    assert lib.gc_comm_init_local(hs, 0, 0) == 1
    assert lib.gc_comm_init_local(hs, 9, 0) == 1
    h = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert lib.gc_comm_init(ctypes.byref(h), 2, 2, uid, 0) == 1      # rank >= world
    assert lib.gc_comm_init(ctypes.byref(h), 0, 9, uid, 0) == 1      # world > GC_MAX_RANKS
    assert lib.gc_comm_destroy(None) == 0


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_1606_06025_b200 import partition_edge_balanced
    from paper_1606_06025_b200.dist import broadcast_uid, local_slice
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        uid = broadcast_uid(lambda: bytes(range(128)))        # rank 0's id reaches every rank
        g = wl.rmat(10, 8, seed=3)
        bounds = partition_edge_balanced(g.row_ptr, world)
        b, e = int(bounds[rank]), int(bounds[rank + 1])
        rpl, cil = local_slice(g.row_ptr, g.col_idx, b, e)
        # stand-in for this rank's gc_color_dist output: the oracle's colours of the range
        mine = oracle.sgr(g)[0][b:e]
        parts = [None] * world
        dist.all_gather_object(parts, (b, e, mine.tolist(), int(rpl[-1]), len(cil)))
        q.put((rank, uid, parts, bounds.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_uid_broadcast_and_gather():
    import torch.multiprocessing as mp
    from paper_1606_06025_b200.dist import assemble
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = wl.rmat(10, 8, seed=3)
    for rank, uid, parts, bounds in outs:
        assert uid == bytes(range(128))
        assert [(b, e) for b, e, *_ in parts] == list(zip(bounds[:-1], bounds[1:]))
        assert all(nnz == ncol for *_, nnz, ncol in parts)
        colors = assemble([np.array(c, np.uint32) for _, _, c, _, _ in parts], bounds)
        assert np.array_equal(colors, oracle.sgr(g)[0])


# ---------------------------------------------------------------- GPU: the real kernels

@pytest.fixture(scope="module")
def gcd():
    import torch
    assert torch.cuda.is_available()
    import paper_1606_06025_b200 as gc
    import paper_1606_06025_b200.dist as d
    return gc, d


def _dev(g):
    import torch
    return (torch.from_numpy(np.ascontiguousarray(g.row_ptr)).cuda(),
            torch.from_numpy(np.ascontiguousarray(g.col_idx) if g.m else np.zeros(1, np.int32)).cuda())


def _check_dist(d, g, bounds, policy, **kw):
    # a lost rank fails the test in seconds (the barriers of these small graphs take microseconds)
    kw["tuning"] = dict(kw.get("tuning") or {}, watchdog_ms=20000)
    rp, ci = _dev(g)
    colors, results = d.color_partitioned_local(rp, ci, bounds, policy, trace=True, **kw)
    ref, nc, r, tr = oracle.sgr(g, policy, trace=True)
    if not np.array_equal(colors, ref):
        bad = np.nonzero(colors != ref)[0]
        raise AssertionError(f"{g.name} {policy} bounds={list(bounds)} {kw}: {len(bad)} mismatches, "
                             f"first v={bad[0]} gpu={colors[bad[0]]} oracle={ref[bad[0]]}")
    for res in results:
        assert res.num_colors == nc and res.rounds == r, (res.num_colors, nc, res.rounds, r)
        assert res.trace == tr
    return results


DIST_GRAPHS = [
    lambda: wl.rmat(13, 8, seed=4), lambda: wl.mesh2d(64, 48, 0.3), lambda: wl.complete(40),
    lambda: wl.star(300, center_last=True), lambda: wl.stencil27(9, 7, 5), lambda: wl.rmat(12, 16, wl.GRAPH500, 3),
    lambda: wl.disjoint_union(wl.rmat(10, 8), wl.star(3000, center_last=True), wl.path(77)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("policy", POLICIES)
def test_gpu_dist_edge_balanced(gcd, parts, policy):
    """Edge-balanced ranges, every policy: bit-identical to the oracle (and so to one GPU)."""
    gc, d = gcd
    for make in DIST_GRAPHS:
        g = make()
        _check_dist(d, g, gc.partition_edge_balanced(g.row_ptr, parts), policy)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_gpu_dist_random_covers(gcd, seed):
    """Arbitrary covers, including empty and unaligned ranges (dense sweeps straddling ranks)."""
    gc, d = gcd
    for make in DIST_GRAPHS[:5]:
        g = make()
        parts = [2, 3, 5, 8, 4, 7][seed]
        b = random_bounds(g.n, parts, seed)
        for policy in POLICIES:
            _check_dist(d, g, b, policy)


@pytest.mark.gpu
@pytest.mark.parametrize("tuning", [dict(n1=0), dict(n1=2), dict(n1=2, dense_div=1), dict(dense_div=1000000000),
                                    dict(dense_div=1), dict(state_bytes=2), dict(state_bytes=4),
                                    dict(n1=2, state_bytes=2), dict(compact=1), dict(variant=1)],
                         ids=lambda t: ",".join(f"{k}={v}" for k, v in t.items()))
def test_gpu_dist_schedules(gcd, tuning):
    """Every schedule knob (dense/sparse switch, dirty-set rounds with remote marks, state width,
    kernel variant) leaves the multi-rank colouring unchanged."""
    gc, d = gcd
    for make in (DIST_GRAPHS[0], DIST_GRAPHS[1], DIST_GRAPHS[4], lambda: wl.complete(70)):
        g = make()
        for policy in POLICIES:
            _check_dist(d, g, gc.partition_edge_balanced(g.row_ptr, 3), policy, tuning=tuning)
            _check_dist(d, g, random_bounds(g.n, 4, 11), policy, tuning=tuning)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [127, 128, 130])
def test_gpu_dist_state_restart(gcd, k):
    """Colours > 127: every rank stops at the same barrier and restarts with 16-bit words."""
    gc, d = gcd
    g = wl.complete(k)
    res = _check_dist(d, g, np.array([0, 5, 64, k], np.int64), "higher_id")
    assert res[0].num_colors == k


@pytest.mark.gpu
def test_gpu_dist_matches_one_gpu_rmat16(gcd):
    """BASELINE configs[0] (R-MAT s16) on 2/4/8 emulated ranks == gc_color == oracle."""
    import torch
    gc, d = gcd
    g = wl.config_graph("rmat16")
    rp, ci = _dev(g)
    one = gc.color(rp, ci)
    for parts in (2, 4, 8):
        colors, res = d.color_partitioned_local(rp, ci, gc.partition_edge_balanced(g.row_ptr, parts))
        assert np.array_equal(colors, one.colors.cpu().numpy().view(np.uint32))
        assert res[0].rounds == one.rounds and res[0].num_colors == one.num_colors
    assert torch.cuda.is_available()


@pytest.mark.gpu
def test_gpu_dist_comm_reuse_and_host_buffers(gcd):
    """One communicator across calls and graph sizes (window grows, epochs continue); host
    (numpy) inputs and outputs."""
    gc, d = gcd
    comms = d.local_group(3)
    try:
        for g in (wl.rmat(11, 8), wl.rmat(13, 8, seed=2), wl.path(50), wl.rmat(11, 8)):
            b = gc.partition_edge_balanced(g.row_ptr, 3)
            rp, ci = _dev(g)
            colors, _ = d.color_partitioned_local(rp, ci, b, comms=comms)
            assert np.array_equal(colors, oracle.sgr(g)[0])
            colors_h, _ = d.color_partitioned_local(g.row_ptr, g.col_idx, b, comms=comms)
            assert np.array_equal(colors_h, oracle.sgr(g)[0])
    finally:
        for c in comms:
            c.close()


@pytest.mark.gpu
def test_gpu_dist_disagreement_and_errors(gcd):
    """Ranges that do not tile [0, n), or a rank whose rows are invalid: every rank returns the
    error (none is left waiting), and the communicator stays usable."""
    import threading
    gc, d = gcd
    g = wl.rmat(10, 8)
    rp, ci = _dev(g)
    comms = d.local_group(2)
    try:
        errs = [None, None]

        def run(q, b, e, cil):
            rpl, _ = d.local_slice(rp, ci, b, e)
            try:
                d.color_dist(comms[q], g.n, b, e, rpl.contiguous(), cil)
            except gc.GcError as ex:
                errs[q] = ex.status
        # gap between the ranges
        th = [threading.Thread(target=run, args=(0, 0, 100, ci[:int(g.row_ptr[100])].contiguous())),
              threading.Thread(target=run, args=(1, 101, g.n, ci[int(g.row_ptr[101]):].contiguous()))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert errs == [1, 1]
        # rank 1's rows hold an out-of-range id: GC_ERR_INVALID_GRAPH reported everywhere
        errs = [None, None]
        bad = ci[int(g.row_ptr[512]):].clone()
        bad[0] = g.n + 5
        th = [threading.Thread(target=run, args=(0, 0, 512, ci[:int(g.row_ptr[512])].contiguous())),
              threading.Thread(target=run, args=(1, 512, g.n, bad))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert errs == [2, 2]
        colors, _ = d.color_partitioned_local(rp, ci, [0, 512, g.n], comms=comms)
        assert np.array_equal(colors, oracle.sgr(g)[0])
    finally:
        for c in comms:
            c.close()
