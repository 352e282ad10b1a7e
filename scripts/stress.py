"""Repeat colourings and require identical output (the result is schedule independent)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1606_06025_b200 as gc, workloads as wl
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for cfg in ("rmat24", "stencil128", "mesh8192", "rmat16"):
    g = wl.config_graph(cfg)
    rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
    for pol in ("higher_id", "lower_id", "degree"):
        ref = gc.color(rp, ci, policy=pol, validate=False).colors.clone()
        assert gc.verify(rp, ci, ref) == -1
        bad = sum(0 if torch.equal(gc.color(rp, ci, policy=pol, validate=False).colors, ref) else 1 for _ in range(reps))
        print(cfg, pol, "repeats", reps, "mismatches", bad, flush=True)
        assert bad == 0
