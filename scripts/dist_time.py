import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads as wl, paper_1606_06025_b200 as gc
from paper_1606_06025_b200.dist import color_partitioned
cfg = sys.argv[1]
g = wl.config_graph(cfg)
rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
ref = gc.color(rp, ci, validate=False)
for parts in (1, 2):
    color_partitioned(rp, ci, parts)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    c, nc, r = color_partitioned(rp, ci, parts)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(cfg, "parts", parts, "%.1f ms" % (dt * 1e3), "rounds", r, "same", bool(torch.equal(c.cuda(), ref.colors)), flush=True)
