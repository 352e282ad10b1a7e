#!/usr/bin/env python
"""Oracle results for the N4 experiment graphs -> tests/golden/n4_oracle.json.

Calls ONLY oracle/ (oracle_sgr and oracle_greedy_alg1) and the
seeded generators: per graph and policy the oracle's rounds, colours and colour-array SHA-256,
and per graph the colours of the sequential greedy Alg. 1 in ascending id order (the paper's
"Serial" analogue for Fig. 7).  scripts/experiments.py compares the GPU runs with these.
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from n4_graphs import graphs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "n4_oracle.json")


def sha(c):
    return hashlib.sha256(np.ascontiguousarray(c, dtype="<u4").tobytes()).hexdigest()


def main():
    rec = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for tags, key, mk, policies, extra in graphs():
        if key in rec and all(p in rec[key]["sgr"] for p in policies):
            continue
        g = mk()
        t0 = time.perf_counter()
        a1, a1n = oracle.greedy_alg1(g)
        ent = {"n": g.n, "m": g.m, "alg1_colors": int(a1n), "alg1_seconds": round(time.perf_counter() - t0, 3),
               "sgr": {}}
        for pol in policies:
            t0 = time.perf_counter()
            c, nc, r = oracle.sgr(g, pol)
            ent["sgr"][pol] = {"colors": int(nc), "rounds": int(r), "sha256_colors_u32le": sha(c),
                               "oracle_seconds": round(time.perf_counter() - t0, 3)}
        rec[key] = ent
        with open(OUT, "w") as f:
            json.dump(rec, f, indent=1)
        print(key, json.dumps(ent["sgr"]), "alg1", a1n, flush=True)


if __name__ == "__main__":
    main()
