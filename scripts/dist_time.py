"""Time the multi-GPU kernels in the one-process emulation (all ranks on one GPU; diagnostics,
not a scaling number): per P, the slowest rank's kernel time of gc_color_dist and whether the
colours equal one-GPU gc_color's.

    python scripts/dist_time.py rmat24 [P ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_06025_b200 as gc  # noqa: E402
import paper_1606_06025_b200.dist as d  # noqa: E402
import workloads as wl  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
parts_list = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
g = wl.config_graph(cfg)
rp = torch.from_numpy(g.row_ptr).cuda()
ci = torch.from_numpy(g.col_idx).cuda()
one = gc.color(rp, ci, validate=False, time_kernel=True)
ref = one.colors.cpu().numpy().view(np.uint32)
print(cfg, "1 GPU gc_color kernel %.2f ms" % one.kernel_ms, flush=True)
for parts in parts_list:
    bounds = gc.partition_edge_balanced(g.row_ptr, parts)
    comms = d.local_group(parts)
    for rep in range(3):
        colors, res = d.color_partitioned_local(rp, ci, bounds, comms=comms, validate=False, time_kernel=True)
        print(cfg, "P", parts, "rep", rep, "slowest rank kernel %.2f ms" % max(r.kernel_ms for r in res),
              "rounds", res[0].rounds, "same", bool(np.array_equal(colors, ref)), flush=True)
    for c in comms:
        c.close()
