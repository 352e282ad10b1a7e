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
