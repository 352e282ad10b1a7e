import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads as wl, paper_1606_06025_b200 as gc
from paper_1606_06025_b200.dist import CudaPartition, LocalComm, local_slice, run_rounds
cfg = sys.argv[1]
g = wl.config_graph(cfg)
rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
ref = gc.color(rp, ci, validate=False)
for parts in (1, 2):
    for rep in range(2):
        bounds = gc.partition_edge_balanced(g.row_ptr, parts)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        objs = []
        for k in range(parts):
            b, e = int(bounds[k]), int(bounds[k + 1])
            rpl, cil = local_slice(rp, ci, b, e)
            objs.append(CudaPartition(g.n, b, e, rpl.contiguous(), cil.contiguous()))
        torch.cuda.synchronize(); t1 = time.perf_counter()
        res = run_rounds(objs, LocalComm())
        torch.cuda.synchronize(); t2 = time.perf_counter()
        c = torch.cat(res.colors_local)
        for o in objs:
            o.close()
        torch.cuda.synchronize(); t3 = time.perf_counter()
        print(cfg, "parts", parts, "create %.1f ms rounds %.1f ms close %.1f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3),
              "rounds", res.rounds, "same", bool(torch.equal(c.cuda(), ref.colors)), flush=True)
