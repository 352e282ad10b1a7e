"""Input generators (workloads/): canonical CSR contract and determinism."""
import numpy as np
import pytest

import workloads as wl


def _canonical(g):
    rp, ci = g.row_ptr, g.col_idx
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == len(ci)
    src = np.repeat(np.arange(g.n), np.diff(rp))
    assert np.all((ci >= 0) & (ci < g.n))
    assert not np.any(ci == src)                                  # no self loops
    same_row = src[1:] == src[:-1]
    assert np.all(ci[1:][same_row] > ci[:-1][same_row])           # sorted, deduplicated
    fwd = set(zip(src.tolist(), ci.tolist()))
    assert all((w, v) in fwd for v, w in fwd)                     # symmetric


def test_spec_csr_examples():
    g = wl.from_edges(3, [(0, 1), (1, 2), (2, 0)])
    assert g.row_ptr.tolist() == [0, 2, 4, 6] and g.col_idx.tolist() == [1, 2, 0, 2, 0, 1]
    g = wl.from_edges(3, [(0, 1), (1, 2)])
    assert g.row_ptr.tolist() == [0, 1, 3, 4] and g.col_idx.tolist() == [1, 0, 2, 1]
    g = wl.from_edges(3, [(0, 1), (1, 0), (2, 2), (0, 1)])
    assert g.col_idx.tolist() == [1, 0]
    with pytest.raises(ValueError):
        wl.from_edges(3, [(0, 5)])


def test_degree_stats_examples():
    s = wl.degree_stats(wl.star(3))
    assert (s["min"], s["max"], s["avg"], s["var"]) == (1, 3, 1.5, 0.75)
    s = wl.degree_stats(wl.path(3))
    assert abs(s["avg"] - 4 / 3) < 1e-12 and abs(s["var"] - 2 / 9) < 1e-12


@pytest.mark.parametrize("make", [lambda: wl.rmat(12, 8), lambda: wl.rmat(10, 16, wl.RMAT_ER, 3),
                                  lambda: wl.stencil27(7, 5, 3), lambda: wl.mesh2d(33, 17, 0.3),
                                  lambda: wl.gnp(50, 0.2, 1)])
def test_canonical_and_deterministic(make):
    g1, g2 = make(), make()
    _canonical(g1)
    assert np.array_equal(g1.row_ptr, g2.row_ptr) and np.array_equal(g1.col_idx, g2.col_idx)


def test_rmat_skew_ordering():
    """Table 1: rmat-g has far larger degree variance than rmat-er."""
    g = wl.rmat(16, 5, wl.RMAT_G)
    e = wl.rmat(16, 5, wl.RMAT_ER)
    assert wl.degree_stats(g)["var"] > 5 * wl.degree_stats(e)["var"]
    assert abs(wl.degree_stats(e)["avg"] - 10) < 0.5


def test_mesh_deletion_fraction():
    g = wl.mesh2d(256, 256, 0.3)
    full = 2 * (2 * 256 * 255)
    assert abs(g.m / full - 0.7) < 0.01 and g.max_degree() <= 4


def test_splitmix64_reference_value():
    # first output of SplitMix64 seeded with 0 (Vigna's reference: x += golden gamma, mix)
    assert wl.splitmix64(0) == 0xE220A8397B1DCDAF


def _rmat_python(scale, ef, abc, seed):
    """Plain-Python transcription of the W1 recipe for tiny scales."""
    M = (1 << 64) - 1

    def sm(x):
        z = (x + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    a, b, c = abc
    n = 1 << scale
    pi = list(range(n))
    for i in range(n - 1, 0, -1):
        j = sm((seed ^ 0x5851F42D4C957F2D) + (n - 1 - i)) % (i + 1)
        pi[i], pi[j] = pi[j], pi[i]
    adj = [set() for _ in range(n)]
    for i in range(ef * n):
        u = v = 0
        for l in range(scale):
            r = (sm(((seed << 40) + 64 * i + l) & M) >> 11) * 2.0 ** -53
            bu, bv = (0, 0) if r < a else (0, 1) if r < a + b else (1, 0) if r < a + b + c else (1, 1)
            u, v = (u << 1) | bu, (v << 1) | bv
        pu, pv = pi[u], pi[v]
        if pu != pv:
            adj[pu].add(pv)
            adj[pv].add(pu)
    return adj


@pytest.mark.parametrize("abc,seed", [(wl.RMAT_G, 1), (wl.GRAPH500, 7)])
def test_rmat_matches_python_recipe(abc, seed):
    g = wl.rmat(7, 8, abc, seed)
    adj = _rmat_python(7, 8, abc, seed)
    for v in range(g.n):
        assert g.adj(v).tolist() == sorted(adj[v])


@pytest.mark.parametrize("bounds", [[0, 1000, 2500, 4096], [0, 0, 17, 4095, 4096], [0, 4096]])
def test_rmat_range_equals_whole_graph(bounds):
    """Rows generated per vertex range (multi-GPU ranks, scale 27) equal the whole graph's."""
    g = wl.rmat(12, 16)
    for b, e in zip(bounds[:-1], bounds[1:]):
        rp, ci = wl.rmat_range(12, 16, b, e)
        assert np.array_equal(rp, g.row_ptr[b:e + 1] - g.row_ptr[b])
        assert np.array_equal(ci, g.col_idx[g.row_ptr[b]:g.row_ptr[e]])


@pytest.mark.gpu
@pytest.mark.parametrize("scale,ef,abc,seed", [(10, 8, wl.RMAT_G, 1), (12, 16, wl.RMAT_G, 1), (11, 16, wl.GRAPH500, 5),
                                               (14, 8, wl.RMAT_ER, 3)])
def test_rmat_range_gpu_equals_cpu(scale, ef, abc, seed):
    """The GPU generator (gen_gpu.cu) builds exactly gen.c's rows, for any range and chunking."""
    n = 1 << scale
    for (b, e), chunk in (((0, n), 1 << 29), ((0, n), 997), ((n // 3, n - 5), 4096), ((7, 7), 1 << 20)):
        rp, ci = wl.rmat_range(scale, ef, b, e, abc, seed)
        rpg, cig = wl.rmat_range_gpu(scale, ef, b, e, abc, seed, chunk_arcs=chunk)
        assert np.array_equal(rpg.cpu().numpy(), rp) and np.array_equal(cig.cpu().numpy(), ci), (b, e, chunk)
