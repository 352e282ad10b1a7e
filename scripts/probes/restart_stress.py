"""Stress: repeated multi-rank colourings of K_130 (8-bit -> 16-bit restart) in the one-GPU
emulation, and variants, reporting every failure (diagnostics for the dist launch path)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1606_06025_b200 as gc, paper_1606_06025_b200.dist as d, workloads as wl, oracle
g = wl.complete(130)
rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
ref = oracle.sgr(g)[0]
iters = int(sys.argv[1])
for name, bounds, tun in (("1-gpu", None, {}), ("P1", [0, 130], {}), ("P2", [0, 64, 130], {}), ("P3", [0, 5, 64, 130], {}),
                          ("P3-u16", [0, 5, 64, 130], dict(state_bytes=2)), ("P3-n1=0", [0, 5, 64, 130], dict(n1=0))):
    fails = 0
    for it in range(iters):
        try:
            if bounds is None:
                c = gc.color(rp, ci, tuning=dict(watchdog_ms=3000)).colors.cpu().numpy().view(np.uint32)
            else:
                c, res = d.color_partitioned_local(rp, ci, np.array(bounds), tuning=dict(tun, watchdog_ms=3000))
            assert np.array_equal(c, ref)
        except Exception as ex:
            fails += 1
            if fails <= 2: print(name, "iter", it, str(ex)[:700], flush=True)
    print(name, "fails", fails, "of", iters, flush=True)
