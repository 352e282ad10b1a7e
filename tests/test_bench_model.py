"""Host-side measurement logic of bench.py (no GPU): the algorithmic-byte models are the
per-unit tables of DESIGN.md §5.3 / SURVEY §8(d) applied to the work counters."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


WORK = dict(phase_a_vertices=30, phase_a_edges=2, phase_b_vertices=40, phase_b_edges=100,
            commit_scatter=200, pushes=5, dense_a_swept=0, dense_b_swept=10,
            sparse_a_entries=20, sparse_b_entries=30, state_bytes=1, pending_degree_sum=300)


def test_design_bytes_per_unit_table():
    b = _bench()
    n = 10
    sw = 1
    expect = ((8 + 4 + sw + 1 + 32) * n                 # ingest
              + (sw + 1) * 0 + 17 * 20 + sw * 30 + (4 + sw) * 2   # Phase A
              + sw * 10 + 12 * (40 - 30) + (16 + sw) * 30         # Phase B sweeps / entries
              + (4 + sw) * 100 + sw * n + 16 * 5 + 8 * 200        # scans, commits, pushes, scatter
              + (sw + 4) * n)                                      # finalize
    assert b.algorithmic_bytes(WORK, n) == expect


def test_design_bytes_counts_issued_scatter_edges():
    """Scatter edges skipped by the commit filter (neighbour seen committed) cost nothing."""
    b = _bench()
    n = 10
    assert b.algorithmic_bytes(dict(WORK, scatter_reds=120), n) == b.algorithmic_bytes(WORK, n) - 8 * 80


def test_survey_bytes_pull_model():
    """sum_{v in W_r} (24 + 8 deg) + sum (28 + 8 s_B), round 1 contributing m."""
    b = _bench()
    n, m = 10, 64
    assert b.survey_bytes(WORK, n, m) == (24 + 28) * 40 + 8 * (m + 300) + 8 * 100


def test_survey_bytes_single_round_edgeless():
    """Edgeless graph: one round, W_1 = V, no neighbours: 52 bytes per vertex."""
    b = _bench()
    w = dict(WORK, phase_b_vertices=7, phase_b_edges=0, pending_degree_sum=0)
    assert b.survey_bytes(w, 7, 0) == 52 * 7
