#!/usr/bin/env python
"""Diagnostics (GPU box): where the time of one gc_color call goes outside the kernel.
Per call: host wall time, torch-event time on the call's stream, the library's kernel time."""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mesh8192")
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    import torch
    import paper_1606_06025_b200 as gc
    import workloads as wl
    g = wl.config_graph(args.config)
    rp = torch.from_numpy(g.row_ptr).cuda()
    ci = torch.from_numpy(g.col_idx).cuda()
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
    for variant in ({}, {"tuning": {"n1": 0}}, {"validate": True}):
        kw = dict(validate=False, out=out)
        kw.update(variant)
        gc.color(rp, ci, **kw)
        torch.cuda.synchronize()
        wall, ev, kms = [], [], []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            r = gc.color(rp, ci, time_kernel=True, **kw)
            e1.record()
            torch.cuda.synchronize()
            wall.append(1e3 * (time.perf_counter() - t0))
            ev.append(e0.elapsed_time(e1))
            kms.append(r.kernel_ms)
        print(args.config, variant, "wall %.3f  stream-events %.3f  kernel %.3f ms" %
              (statistics.median(wall), statistics.median(ev), statistics.median(kms)), flush=True)


if __name__ == "__main__":
    main()
