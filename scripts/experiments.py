#!/usr/bin/env python
"""the paper's measurement dimensions re-run on synthetic graphs with the
finished GPU path (no comparison systems, no UF matrices).  GPU only; prints JSON lines.

  fig4  : rounds (iterations) and colours under the id policy vs the degree heuristic
          (Fig. 4) on rmat-er / rmat-g at 1M vertices, d = 10, a 27-point
          stencil and a 2-D mesh;
  fig9  : rmat-er scale sweep 2^19 .. 2^24 at d = 10 (Fig. 9);
  fig10 : rmat-er density sweep at 2^20 vertices, d = 2 .. 80 (Fig. 10).
d = directed entries per vertex (Table 1 convention, reading C15): edge factor = d / 2.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="fig4,fig9,fig10")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_1606_06025_b200 as gc
    import workloads as wl

    def run(exp, g, policy, **extra):
        rp = torch.from_numpy(g.row_ptr).cuda()
        ci = torch.from_numpy(g.col_idx).cuda()
        res = gc.color(rp, ci, policy=policy, validate=True)
        ok = gc.verify(rp, ci, res.colors) == -1
        ts = [gc.color(rp, ci, policy=policy, validate=False, time_kernel=True).kernel_ms for _ in range(args.reps)]
        ms = statistics.median(ts)
        line = {"exp": exp, "graph": g.name, "n": g.n, "m": g.m, "policy": policy, "rounds": res.rounds,
                "colors": res.num_colors, "kernel_ms": round(ms, 4), "gteps": round(g.m / ms / 1e6, 3),
                "verified": ok, **extra}
        print(json.dumps(line), flush=True)

    only = set(args.only.split(","))
    if "fig4" in only:
        graphs = [wl.rmat(20, 5, wl.RMAT_ER), wl.rmat(20, 5, wl.RMAT_G), wl.rmat(20, 16, wl.GRAPH500),
                  wl.stencil27(64), wl.mesh2d(2048, 2048, 0.3), wl.config_graph("rmat24")]
        for g in graphs:
            for pol in ("higher_id", "lower_id", "degree"):
                run("fig4", g, pol)
    if "fig9" in only:
        for sc in range(19, 25):
            g = wl.rmat(sc, 5, wl.RMAT_ER)
            for pol in ("higher_id", "degree"):
                run("fig9", g, pol, scale=sc, avg_degree=2 * 5)
    if "fig10" in only:
        for ef in (1, 2, 5, 10, 20, 40):
            g = wl.rmat(20, ef, wl.RMAT_ER)
            for pol in ("higher_id", "degree"):
                run("fig10", g, pol, scale=20, avg_degree=2 * ef)


if __name__ == "__main__":
    main()
