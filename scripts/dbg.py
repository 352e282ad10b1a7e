import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1606_06025_b200 as gc, workloads as wl, oracle
g = wl.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 16, 8)
rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
kw = eval(sys.argv[2]) if len(sys.argv) > 2 else {}
try:
    r = gc.color(rp, ci, **kw)
    c = r.colors.cpu().numpy().view(np.uint32)
    ref = oracle.sgr(g)[0]
    print("ok", r.rounds, np.array_equal(c, ref))
except Exception as e:
    print("ERR", e)
