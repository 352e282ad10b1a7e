"""The synthetic graphs of SURVEY §8(f) N4 (the paper's measurement dimensions on synthetic
inputs): one list shared by scripts/make_n4_goldens.py (CPU oracle) and scripts/experiments.py
(GPU).  d = directed entries per vertex (Table 1 convention, reading C15): edge factor = d / 2.

  fig4  : iterations and colours under the id policies vs the degree heuristic
  fig7  : colours of the parallel method vs the sequential greedy Alg. 1
  fig9  : rmat-er scale sweep 2^19 .. 2^24 at d = 10
  fig10 : rmat-er density sweep at 2^20 vertices, d = 2 .. 80
"""
import workloads as wl


def graphs():
    """(experiment tags, key, builder, policies, extra fields)"""
    out = []
    fig47 = [("rmat-er s20 d10", lambda: wl.rmat(20, 5, wl.RMAT_ER)),
             ("rmat-g s20 d10", lambda: wl.rmat(20, 5, wl.RMAT_G)),
             ("graph500 s20 d32", lambda: wl.rmat(20, 16, wl.GRAPH500)),
             ("stencil27 64^3", lambda: wl.stencil27(64)),
             ("mesh 2048^2 30% deleted", lambda: wl.mesh2d(2048, 2048, 0.3)),
             ("rmat-g s24 d32 (configs[2])", lambda: wl.config_graph("rmat24"))]
    for key, mk in fig47:
        out.append((("fig4", "fig7"), key, mk, ("higher_id", "lower_id", "degree"), {}))
    for sc in range(19, 25):
        out.append((("fig9",), f"rmat-er s{sc} d10", (lambda s=sc: wl.rmat(s, 5, wl.RMAT_ER)), ("higher_id", "degree"),
                    {"scale": sc, "avg_degree": 10}))
    for ef in (1, 2, 5, 10, 20, 40):
        if ef == 5:
            continue  # = fig9's s20 point and fig4's rmat-er s20 d10
        out.append((("fig10",), f"rmat-er s20 d{2 * ef}", (lambda e=ef: wl.rmat(20, e, wl.RMAT_ER)),
                    ("higher_id", "degree"), {"scale": 20, "avg_degree": 2 * ef}))
    return out
