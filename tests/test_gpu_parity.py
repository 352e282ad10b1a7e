"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar: bit-exact colours, identical num_colors, rounds and |W_r| trace —
everything here is integer work.  Inputs are the seeded generators of workloads/.
"""
import numpy as np
import pytest

import oracle
import workloads as wl

pytestmark = pytest.mark.gpu

POLICIES = ["higher_id", "lower_id", "degree"]


@pytest.fixture(scope="module")
def gc():
    import torch
    assert torch.cuda.is_available()
    import paper_1606_06025_b200 as gc
    return gc


def _dev(g):
    import torch
    return (torch.from_numpy(np.ascontiguousarray(g.row_ptr)).cuda(),
            torch.from_numpy(np.ascontiguousarray(g.col_idx) if g.m else np.zeros(1, np.int32)).cuda())


def _gpu_colors(res):
    c = res.colors
    if hasattr(c, "cpu"):
        c = c.cpu().numpy().view(np.uint32)
    return np.asarray(c, dtype=np.uint32)


def _check(gc, g, policy="higher_id", **kw):
    rp, ci = _dev(g)
    res = gc.color(rp, ci, policy=policy, trace=True, **kw)
    c_ref, nc_ref, r_ref, tr_ref = oracle.sgr(g, policy, trace=True)
    c = _gpu_colors(res)
    if not np.array_equal(c, c_ref):
        bad = np.nonzero(c != c_ref)[0]
        raise AssertionError(f"{g.name} {policy} {kw}: {len(bad)} mismatches, first v={bad[0]} "
                             f"gpu={c[bad[0]]} oracle={c_ref[bad[0]]}")
    assert res.num_colors == nc_ref and res.rounds == r_ref, (res.num_colors, nc_ref, res.rounds, r_ref)
    assert res.trace == tr_ref
    return res


SMALL = [
    lambda: wl.cycle(5), lambda: wl.path(4), lambda: wl.path(1000), lambda: wl.complete(33),
    lambda: wl.complete(65), lambda: wl.star(5000), lambda: wl.star(5000, center_last=True),
    lambda: wl.mesh2d(64, 64), lambda: wl.mesh2d(100, 77, 0.3), lambda: wl.stencil27(9, 7, 5),
    lambda: wl.gnp(300, 0.05, 1), lambda: wl.gnp(200, 0.3, 2), lambda: wl.rmat(12, 8),
    lambda: wl.rmat(12, 16, wl.GRAPH500, 3), lambda: wl.edgeless(1), lambda: wl.edgeless(1000),
    lambda: wl.disjoint_union(wl.complete(40), wl.path(7), wl.edgeless(3), wl.star(300)),
    lambda: wl.star(40000), lambda: wl.disjoint_union(wl.rmat(10, 8), wl.star(33000, center_last=True)),
]


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("make", SMALL, ids=range(len(SMALL)))
def test_parity_small(gc, make, policy):
    _check(gc, make(), policy)


@pytest.mark.parametrize("policy", POLICIES)
def test_parity_rmat16_config0(gc, policy):
    """BASELINE.json configs[0]: R-MAT scale 16, edge factor 8, 1 GPU vs CPU oracle."""
    _check(gc, wl.config_graph("rmat16"), policy)


@pytest.mark.parametrize("kw", [
    dict(pull_firstfit=True), dict(host_rounds=True), dict(host_rounds=True, pull_firstfit=True),
    dict(thread_bin_max=1, warp_bin_max=2), dict(thread_bin_max=64, warp_bin_max=64),
    dict(thread_bin_max=1, warp_bin_max=1), dict(blocks_per_sm=1), dict(validate=False),
    dict(count_work=True), dict(symmetry=True),
])
def test_parity_variants(gc, kw):
    """Every launch geometry / driver / First-Fit variant gives the same result (C2, C12)."""
    for g in (wl.rmat(13, 8, seed=7), wl.rmat(11, 16, wl.GRAPH500, 5), wl.complete(70)):
        for pol in POLICIES:
            _check(gc, g, pol, **kw)


TUNINGS = [dict(state_bytes=2), dict(state_bytes=4), dict(scatter_filter=1),
           dict(dense_div=0), dict(dense_div=1), dict(dense_div=1000000000), dict(n1=0), dict(n1=2),
           dict(n1=2, dense_div=1), dict(n1=2, dense_div=1000000000), dict(n1=2, state_bytes=2),
           dict(list=0), dict(list=2), dict(list=2, n1=2), dict(list=2, dense_div=1), dict(compact=1),
           dict(compact=1, n1=0), dict(variant=1), dict(variant=1, n1=2, dense_div=1), dict(variant=0),
           dict(dch=2), dict(n1_chg=4), dict(dense_div=4, dense_div_n1=64)]


def _tid(t):
    return ",".join(f"{k}={v}" for k, v in t.items())


@pytest.mark.parametrize("tuning", TUNINGS, ids=_tid)
def test_parity_tuning_variants(gc, tuning):
    """Every schedule knob of gc_tuning (forced state widths, dense/sparse switch, dirty-set
    and list rounds, filtered commit scatter, kernel variant): same result."""
    for g in (wl.rmat(13, 8, seed=7), wl.rmat(11, 16, wl.GRAPH500, 5), wl.complete(70), wl.complete(130),
              wl.disjoint_union(wl.star(3000), wl.mesh2d(40, 30, 0.3), wl.star(2000, center_last=True)),
              wl.stencil27(9, 7, 5)):
        for pol in POLICIES:
            _check(gc, g, pol, tuning=tuning)
            _check(gc, g, pol, warp_bin_max=8, tuning=tuning)
        _check(gc, g, "higher_id", host_rounds=True, tuning=tuning)


@pytest.mark.parametrize("tuning", [dict(list=2), dict(list=2, n1=2), dict(list=2, dense_div=1),
                                    dict(list=2, dense_div=0), dict(list=1)], ids=_tid)
def test_parity_list_rounds(gc, tuning):
    """List rounds (bounded degree <= 64, 8-bit words): entered from dense, sparse or switch rounds."""
    for g in (wl.mesh2d(100, 77, 0.3), wl.mesh2d(64, 64), wl.stencil27(9, 7, 5), wl.stencil27(12),
              wl.gnp(400, 0.02, 3), wl.path(1000), wl.cycle(999), wl.rmat(12, 2, wl.RMAT_ER)):
        assert g.max_degree() <= 64
        for pol in POLICIES:
            _check(gc, g, pol, tuning=tuning)


def test_bad_tuning_rejected(gc):
    rp, ci = _dev(wl.path(10))
    with pytest.raises(gc.GcError) as e:
        gc.color(rp, ci, tuning=dict(state_bytes=3))
    assert e.value.status == 1


@pytest.mark.parametrize("tuning", [{}, dict(widen=0), dict(dense_div=1000000000), dict(dense_div=0),
                                    dict(n1=2, dense_div=1000000000)], ids=_tid)
@pytest.mark.parametrize("k", [126, 127, 128, 129, 136])
def test_state_word_restart(gc, k, tuning):
    """8-bit state words hold colours <= 127: K_k needs colour k, so from K_128 on the run stops
    at the Phase A that overflows and goes on with 16-bit words — widened in place and resumed
    there (default, in a dense or a sparse round), or restarted (widen=0); colours up to 512 come
    from the 64 forbidden-colour planes, beyond from the windowed fallback (reading C7)."""
    res = _check(gc, wl.complete(k), tuning=tuning)
    assert res.num_colors == k


@pytest.mark.parametrize("tuning", [{}, dict(widen=0)], ids=_tid)
def test_widen_graph500(gc, tuning):
    """Graph500-skew R-MAT with > 127 colours: 8 -> 16-bit widening in place vs restart."""
    res = _check(gc, wl.rmat(15, 32, wl.GRAPH500, 1), tuning=tuning)  # 136 colours, max degree 8673
    assert res.num_colors > 127


def test_multiwindow_colors(gc):
    """K_1025 and Graph500 skew: colours far beyond the 32-bit mask and 64-bit windows (C7)."""
    _check(gc, wl.complete(300))
    g = wl.rmat(14, 16, wl.GRAPH500, 1)
    res = _check(gc, g)
    assert res.num_colors > 64


@pytest.mark.slow
def test_complete_1025(gc):
    _check(gc, wl.complete(1025), thread_bin_max=16, warp_bin_max=256)


def test_host_buffers(gc):
    """Host (numpy) inputs and output: the library copies in and out (e2e path)."""
    g = wl.rmat(12, 8, seed=9)
    res = gc.color(g.row_ptr, g.col_idx)
    c_ref, nc, r = oracle.sgr(g)
    assert np.array_equal(np.asarray(res.colors), c_ref) and res.rounds == r


def test_degenerate(gc):
    import torch
    res = gc.color(torch.zeros(1, dtype=torch.int64, device="cuda"), torch.zeros(1, dtype=torch.int32, device="cuda"))
    assert res.num_colors == 0 and res.rounds == 0
    _check(gc, wl.edgeless(1))


def test_no_convergence(gc):
    rp, ci = _dev(wl.complete(20))
    with pytest.raises(gc.GcError) as e:
        gc.color(rp, ci, max_rounds=19)
    assert e.value.status == 3
    for host_rounds in (False, True):
        assert gc.color(rp, ci, max_rounds=20, host_rounds=host_rounds).rounds == 20


@pytest.mark.parametrize("bad", ["self", "order", "range", "dup", "asym", "rowptr"])
def test_validation_errors(gc, bad):
    import torch
    g = wl.path(6)
    rp, ci = g.row_ptr.copy(), g.col_idx.copy()
    sym = False
    if bad == "self":
        ci[0] = 0
    elif bad == "order":
        ci[1], ci[2] = ci[2], ci[1]
    elif bad == "range":
        ci[3] = 99
    elif bad == "dup":
        ci[2] = ci[1]
    elif bad == "asym":
        ci[-1] = 3  # vertex 5's only neighbour becomes 3 (3 does not list 5)
        sym = True
    elif bad == "rowptr":
        rp[3] = rp[2] - 1
    with pytest.raises(gc.GcError) as e:
        gc.color(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), symmetry=sym)
    assert e.value.status == 2


def test_device_verifier(gc):
    import torch
    g = wl.rmat(12, 8)
    rp, ci = _dev(g)
    res = gc.color(rp, ci)
    assert gc.verify(rp, ci, res.colors) == -1
    bad = res.colors.clone()
    bad[5] = bad[5] + 1
    assert gc.verify(rp, ci, bad) >= 0
    c_alg1, _ = oracle.greedy_alg1(g)
    assert gc.verify(rp, ci, torch.from_numpy(c_alg1.view(np.int32)).cuda()) == -1


def test_determinism_repeat(gc):
    g = wl.rmat(15, 16, seed=2)
    rp, ci = _dev(g)
    first = _gpu_colors(gc.color(rp, ci))
    for _ in range(5):
        assert np.array_equal(_gpu_colors(gc.color(rp, ci)), first)


def test_stencil128_config1_closed_form(gc):
    """BASELINE.json configs[1] at full size: pin P6 (8 colours, 197 rounds, parity formula)."""
    import torch
    g = wl.config_graph("stencil128")
    rp, ci = _dev(g)
    res = gc.color(rp, ci)
    ids = torch.arange(g.n, device="cuda")
    x, y, z = ids % 128, (ids // 128) % 128, ids // (128 * 128)
    expect = (1 + (x % 2) + 2 * (y % 2) + 4 * (z % 2)).to(torch.int32)
    assert torch.equal(res.colors, expect)
    assert res.num_colors == 8 and res.rounds == 197
