#!/usr/bin/env python
"""the paper's measurement dimensions re-run on synthetic graphs with the
finished GPU path (no comparison systems, no UF matrices).  GPU only; prints JSON lines.

Graphs and tags: scripts/n4_graphs.py (fig4 rounds/colours by policy; fig7
colours vs the sequential greedy Alg. 1; fig9 rmat-er scale sweep,
PAPER.md:924-951; fig10 rmat-er density sweep).  Every colouring is compared
with the CPU oracle's result stored in tests/golden/n4_oracle.json (scripts/make_n4_goldens.py,
oracle only): `oracle_match` = same colour-array SHA-256, colours and rounds; `alg1_colors` is
Alg. 1's colour count on the same graph.

    python scripts/experiments.py [--only fig4,fig7,fig9,fig10] > profiles/r02_experiments.jsonl
"""
import argparse
import hashlib
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="fig4,fig7,fig9,fig10")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1606_06025_b200 as gc
    from n4_graphs import graphs

    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "n4_oracle.json")))
    only = set(args.only.split(","))
    for tags, key, mk, policies, extra in graphs():
        tags = [t for t in tags if t in only]
        if not tags:
            continue
        g = mk()
        rp = torch.from_numpy(g.row_ptr).cuda()
        ci = torch.from_numpy(g.col_idx).cuda()
        gk = gold.get(key)
        for pol in policies:
            res = gc.color(rp, ci, policy=pol, validate=True)
            c = res.colors.cpu().numpy().view(np.uint32)
            ok = gc.verify(rp, ci, res.colors) == -1
            ts = [gc.color(rp, ci, policy=pol, validate=False, time_kernel=True).kernel_ms for _ in range(args.reps)]
            ms = statistics.median(ts)
            go = gk["sgr"].get(pol) if gk else None
            match = None if go is None else bool(
                hashlib.sha256(np.ascontiguousarray(c, dtype="<u4").tobytes()).hexdigest() == go["sha256_colors_u32le"]
                and res.num_colors == go["colors"] and res.rounds == go["rounds"])
            line = {"exp": "+".join(tags), "graph": key, "n": g.n, "m": g.m, "policy": pol, "rounds": res.rounds,
                    "colors": res.num_colors, "alg1_colors": gk["alg1_colors"] if gk else None,
                    "colors_vs_alg1": round(res.num_colors / gk["alg1_colors"], 4) if gk else None,
                    "kernel_ms": round(ms, 4), "gteps": round(g.m / ms / 1e6, 3), "verified": ok,
                    "oracle_match": match, "oracle_seconds": go["oracle_seconds"] if go else None, **extra}
            print(json.dumps(line), flush=True)
        del rp, ci


if __name__ == "__main__":
    main()
