import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1606_06025_b200 as gc, workloads as wl, oracle
g = {"rmat13": lambda: wl.rmat(13, 8, seed=7), "g500": lambda: wl.rmat(11, 16, wl.GRAPH500, 5),
     "k70": lambda: wl.complete(70), "rmat16": lambda: wl.config_graph("rmat16")}[sys.argv[1]]()
kw = eval(sys.argv[2]) if len(sys.argv) > 2 else {}
rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
for pol in ("higher_id", "lower_id", "degree"):
    res = gc.color(rp, ci, policy=pol, **kw)
    c = res.colors.cpu().numpy().view(np.uint32)
    cr, nc, r = oracle.sgr(g, pol)
    print(sys.argv[1], pol, kw, "ok" if np.array_equal(c, cr) else "MISMATCH", res.rounds, r, flush=True)
