#!/usr/bin/env python
"""Tuning sweeps on the GPU box (not part of the product or the bench contract).

    python scripts/perf.py --config rmat24 --sweep bins
Prints one line per variant: kernel ms (median of --reps), GTEPS, and whether the colours
equal the default run's (they must: the result is schedule independent).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rmat24")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sweep", default="default")
    ap.add_argument("--barrier", action="store_true")
    ap.add_argument("--tuning", default="", help="gc_tuning overrides as JSON (phases sweep)")
    args = ap.parse_args()

    import torch
    import paper_1606_06025_b200 as gc
    import workloads as wl

    if args.barrier:
        for bps in (1, 2, 4, 0):
            print(json.dumps({"barrier_us": gc.bench_grid_sync(0, bps, 2000), "blocks_per_sm": bps}), flush=True)

    g = wl.config_graph(args.config)
    rp = torch.from_numpy(g.row_ptr).cuda()
    ci = torch.from_numpy(g.col_idx).cuda()
    ref = gc.color(rp, ci, validate=False)
    ref_c = ref.colors.clone()

    variants = {"default": [dict()]}
    variants["bins"] = [dict(thread_bin_max=t1, warp_bin_max=t3)
                        for t1 in (16, 32, 64) for t3 in (128, 256, 512, 1024, 4096)]
    variants["grid"] = [dict(blocks_per_sm=b) for b in (1, 2, 3, 4, 5, 6, 8)]
    variants["modes"] = [dict(), dict(pull_firstfit=True), dict(host_rounds=True),
                         dict(host_rounds=True, pull_firstfit=True)]
    variants["policy"] = [dict(policy=p) for p in ("higher_id", "lower_id", "degree")]
    T = lambda **t: dict(tuning=t)  # noqa: E731  (gc_tuning overrides)
    variants["compact"] = [dict(), T(compact=1), T(compact=1, dense_div=16), T(compact=1, dense_div=64)]
    variants["n1chg"] = [dict(), T(n1=0, dense_div=16)] + [T(n1_chg=x) for x in (2, 4, 8, 16)]
    variants["list"] = [T(list=x) for x in (0, 1, 2)]
    variants["n1"] = [T(n1=x) for x in (0, 1, 2)]
    variants["dense"] = [T(dense_div=d) for d in (0, 2, 4, 8, 16, 64)]
    variants["t3"] = [dict(warp_bin_max=t) for t in (512, 768, 1024, 1536, 2048)]
    variants["dch"] = [T(dch=d) for d in (2, 4, 8, 16, 32)]
    variants["div"] = [T(dense_div=d) for d in (2, 3, 4, 6)]
    variants["densen1"] = [T(dense_div=d, n1=2) for d in (4, 8, 16, 32, 64, 256)]
    variants["misc"] = [dict(), T(scatter_filter=1), T(state_bytes=2), T(variant=0), T(variant=1)]
    if args.sweep == "phases":
        kw = dict(tuning=json.loads(args.tuning)) if args.tuning else {}
        res = gc.color(rp, ci, validate=False, phase_times=True, **kw)
        tot = [sum(x[i] for x in res.phase_us) for i in range(4)]
        print(json.dumps({"config": args.config, "rounds": res.rounds, "phaseA_us": round(tot[0], 1),
                          "phaseB_us": round(tot[1], 1), "A_after_last_cta_us": round(tot[2], 1),
                          "B_after_last_cta_us": round(tot[3], 1)}))
        for r, ((a, b, aw, bw), w) in enumerate(zip(res.phase_us, res.trace), 1):
            print(f"  r={r:3d} |W|={w:10d} A={a:8.1f}us (barrier {aw:6.1f})  B={b:8.1f}us (barrier {bw:6.1f})")
        return
    for kw in variants[args.sweep]:
        kw = dict(kw)
        ts = []
        res = None
        for _ in range(args.reps):
            res = gc.color(rp, ci, validate=False, time_kernel=True, **kw)
            ts.append(res.kernel_ms)
        ms = statistics.median(ts)
        same = bool(torch.equal(res.colors, ref_c)) if "policy" not in kw else None
        print(json.dumps({"config": args.config, "kw": kw, "kernel_ms": round(ms, 4),
                          "gteps": round(g.m / ms / 1e6, 3), "rounds": res.rounds,
                          "colors": res.num_colors, "same_as_default": same}), flush=True)


if __name__ == "__main__":
    main()
