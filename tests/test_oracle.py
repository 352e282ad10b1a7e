"""Pins for the CPU oracle (oracle/oracle.c) — each against something other than itself.

P1  exhaustive cross-implementation vs tests/pyref.py on every labelled graph <= 6 vertices
P2  hand-traced worked examples (tests/golden/worked_examples.json)
P3-P8 closed forms (K_n, P_n, R x C grid, 27-point stencil, stars, edgeless/n=0/n=1)
P9-P14 invariants (FF-fixpoint, greedy bounds, rounds >= colours, progress,
        relabel symmetry, brute-force chromatic number)
P15 Alg. 1 examples
Citations and derivations: DESIGN.md "Oracle pins".
"""
import json
import math
import os
from itertools import combinations

import numpy as np
import pytest

import oracle
import workloads as wl
from tests import pyref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")
POLICIES = ["higher_id", "lower_id", "degree"]


def _all_graphs(max_n):
    for n in range(0, max_n + 1):
        pairs = list(combinations(range(n), 2))
        for mask in range(1 << len(pairs)):
            yield n, [pairs[i] for i in range(len(pairs)) if mask >> i & 1]


def _tiny_csr(n, edges):
    adj = [[] for _ in range(n)]
    for u, v in edges:
        adj[u].append(v)
        adj[v].append(u)
    rp = np.zeros(n + 1, dtype=np.int64)
    for v in range(n):
        rp[v + 1] = rp[v] + len(adj[v])
    ci = np.array([w for v in range(n) for w in sorted(adj[v])], dtype=np.int32)
    return wl.Graph(n, rp, ci), [set(a) for a in adj]


# ---------------------------------------------------------------- P1 (exhaustive)

def test_p1_exhaustive_small_graphs_all_policies():
    """C oracle == independent Python transliteration on all 33,867 graphs <= 6 vertices,
    plus invariants P9-P14 on each."""
    count = 0
    for n, edges in _all_graphs(6):
        g, adj = _tiny_csr(n, edges)
        deg = [len(a) for a in adj]
        res = {}
        for pol in POLICIES:
            c, nc, r, tr = oracle.sgr(g, pol, trace=True)
            pc, pnc, pr, ptr = pyref.sgr(n, adj, pol)
            assert list(c) == pc and nc == pnc and r == pr and tr == ptr, (n, edges, pol)
            res[pol] = list(c)
            if n:
                assert oracle.verify(g, c)[0] == 0                      # P9 proper+complete+FF
                assert all(c[v] <= deg[v] + 1 for v in range(n))       # P10
                assert r >= nc                                         # P11
                assert all(tr[i] > tr[i + 1] for i in range(len(tr) - 1))  # P13
                assert r <= n
        # P12 relabel symmetry: LOWER(G)[v] == HIGHER(pi G)[n-1-v]
        rev_edges = [(n - 1 - u, n - 1 - v) for u, v in edges]
        grev, _ = _tiny_csr(n, rev_edges)
        ch, _, _ = oracle.sgr(grev, "higher_id")
        assert res["lower_id"] == [int(ch[n - 1 - v]) for v in range(n)]
        count += 1
    assert count == 33868  # 33,867 non-empty labelled graphs + the empty graph


def test_p14_bruteforce_chromatic_le_colors_exhaustive():
    """chi(G) <= num_colors for every graph <= 6 vertices (BASELINE.json north star)."""
    for n, edges in _all_graphs(6):
        if n == 0:
            continue
        g, adj = _tiny_csr(n, edges)
        chi = oracle.chromatic_bruteforce(g)
        _, nc, _ = oracle.sgr(g)
        assert 1 <= chi <= nc


def test_alg1_exhaustive_vs_python():
    for n, edges in _all_graphs(5):
        g, adj = _tiny_csr(n, edges)
        c, nc = oracle.greedy_alg1(g)
        assert list(c) == pyref.greedy(n, adj)
        if n:
            assert oracle.verify(g, c)[0] == 0


# ---------------------------------------------------------------- P2 worked examples

def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _golden()["cases"], ids=lambda c: f"{c['name']}-{c['policy']}")
def test_p2_worked_examples(case):
    g = wl.from_edges(case["n"], case["edges"] or np.zeros((0, 2), np.int32))
    c, nc, r, tr = oracle.sgr(g, case["policy"], trace=True)
    assert list(c) == case["colors"]
    assert r == case["rounds"]
    assert tr == case["trace"]
    assert nc == max(case["colors"])


@pytest.mark.parametrize("case", _golden()["alg1"], ids=lambda c: c["name"])
def test_p15_alg1_examples(case):
    g = wl.from_edges(case["n"], case["edges"])
    c, nc = oracle.greedy_alg1(g)
    assert nc == case["num_colors"]
    if "colors" in case:
        assert list(c) == case["colors"]


def test_c5_differs_from_alg1():
    """Reading C5/fact 2: Jacobi SGR is not Alg. 1 (smallest counterexample C5)."""
    g = wl.cycle(5)
    assert list(oracle.sgr(g)[0]) != list(oracle.greedy_alg1(g)[0])


# ---------------------------------------------------------------- P3-P8 closed forms

@pytest.mark.parametrize("n", [1, 2, 3, 5, 11, 33, 65])
def test_p3_complete_graph(n):
    c, nc, r = oracle.sgr(wl.complete(n))
    assert list(c) == list(range(1, n + 1)) and nc == n and r == n


@pytest.mark.parametrize("n", [2, 3, 4, 7, 10, 29, 1000])
def test_p4_path(n):
    c, nc, r = oracle.sgr(wl.path(n))
    assert list(c) == [1 + v % 2 for v in range(n)]
    assert r == 1 + math.ceil((n - 1) / 2)


@pytest.mark.parametrize("R,C", [(1, 2), (2, 2), (3, 5), (8, 8), (7, 3), (64, 64)])
def test_p5_grid(R, C):
    c, nc, r = oracle.sgr(wl.mesh2d(R, C))
    assert list(c) == [1 + (i + j) % 2 for i in range(R) for j in range(C)]
    assert r == 1 + math.ceil((R + C - 2) / 2)


@pytest.mark.parametrize("N", list(range(2, 13)) + [32])
def test_p6_stencil27(N):
    """colour = 1 + (x mod 2) + 2(y mod 2) + 4(z mod 2) == Alg. 1; rounds = 8 + 3*floor((N-2)/2)."""
    g = wl.stencil27(N)
    c, nc, r = oracle.sgr(g)
    ids = np.arange(g.n)
    x, y, z = ids % N, (ids // N) % N, ids // (N * N)
    expect = 1 + (x % 2) + 2 * (y % 2) + 4 * (z % 2)
    assert np.array_equal(c, expect.astype(np.uint32))
    assert r == 8 + 3 * ((N - 2) // 2)
    assert np.array_equal(oracle.greedy_alg1(g)[0], c)


def test_p6_stencil27_edge_count_128():
    """m = (3N-2)^3 - N^3 directed entries at N=128."""
    g = wl.stencil27(128)
    assert g.m == 53_645_816 and g.max_degree() == 26


@pytest.mark.parametrize("k", [1, 3, 100, 5000])
def test_p7_star(k):
    c, nc, r = oracle.sgr(wl.star(k))
    assert c[0] == 1 and all(c[1:] == 2) and r == 2
    c, nc, r = oracle.sgr(wl.star(k, center_last=True))
    assert c[k] == 2 and all(c[:k] == 1) and r == 2


def test_p8_degenerate():
    c, nc, r = oracle.sgr(wl.edgeless(0))
    assert len(c) == 0 and nc == 0 and r == 0
    c, nc, r = oracle.sgr(wl.edgeless(1))
    assert list(c) == [1] and nc == 1 and r == 1
    c, nc, r = oracle.sgr(wl.edgeless(1000))
    assert all(c == 1) and r == 1


def test_max_rounds_no_convergence():
    with pytest.raises(oracle.NoConvergence):
        oracle.sgr(wl.complete(10), max_rounds=9)
    assert oracle.sgr(wl.complete(10), max_rounds=10)[2] == 10


# ---------------------------------------------------------------- invariants at scale

@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("policy", POLICIES)
def test_invariants_random(seed, policy):
    for g in (wl.gnp(60, 0.1, seed), wl.rmat(12, 8, seed=seed), wl.mesh2d(40, 40, 0.3, seed)):
        c, nc, r, tr = oracle.sgr(g, policy, trace=True)
        d = g.degrees()
        assert oracle.verify(g, c)[0] == 0
        assert np.all(c <= d + 1) and nc <= g.max_degree() + 1
        assert r >= nc and r <= g.n
        assert all(tr[i] > tr[i + 1] for i in range(len(tr) - 1)) and tr[0] == g.n


def test_relabel_symmetry_rmat():
    g = wl.rmat(12, 8, seed=5)
    lo, _, rl = oracle.sgr(g, "lower_id")
    hi, _, rh = oracle.sgr(wl.relabel_reverse(g), "higher_id")
    assert np.array_equal(lo, hi[::-1]) and rl == rh


@pytest.mark.parametrize("seed", range(6))
def test_p14_bruteforce_random_10(seed):
    g = wl.gnp(10, 0.45, seed)
    chi = oracle.chromatic_bruteforce(g)
    assert chi <= oracle.sgr(g)[1]
    assert chi <= oracle.greedy_alg1(g)[1]


def test_bruteforce_known_values():
    assert oracle.chromatic_bruteforce(wl.complete(6)) == 6
    assert oracle.chromatic_bruteforce(wl.cycle(5)) == 3
    assert oracle.chromatic_bruteforce(wl.cycle(6)) == 2
    assert oracle.chromatic_bruteforce(wl.edgeless(4)) == 1
    petersen = [(i, (i + 1) % 5) for i in range(5)] + [(i, i + 5) for i in range(5)] + \
               [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
    assert oracle.chromatic_bruteforce(wl.from_edges(10, petersen)) == 3


def test_verifier_detects_each_violation():
    g = wl.path(3)
    assert oracle.verify(g, [1, 2, 1]) == (0, -1)
    assert oracle.verify(g, [1, 0, 1])[0] == 1
    assert oracle.verify(g, [1, 1, 2])[0] == 2
    assert oracle.verify(g, [2, 1, 2])[0] == 0
    assert oracle.verify(g, [1, 3, 1]) == (3, 1)      # proper but not First-Fit
    assert oracle.verify(wl.edgeless(2), [1, 2]) == (3, 1)


def test_rmat16_config_invariants():
    """BASELINE.json configs[0]; the oracle output used by the GPU parity tests."""
    g = wl.config_graph("rmat16")
    c, nc, r = oracle.sgr(g)
    assert oracle.verify(g, c)[0] == 0
    assert nc <= g.max_degree() + 1 and r >= nc
    _, n1 = oracle.greedy_alg1(g)
    assert abs(nc - n1) <= max(3, n1 // 2)
