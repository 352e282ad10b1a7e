#!/usr/bin/env python
"""Write oracle goldens for the full-size BASELINE.json configs (tests/golden/oracle_*.json).

Calls ONLY oracle/ (and the seeded generators of workloads/): every stored value is the CPU
oracle's (oracle_sgr, Alg. 7 with the readings C1-C17 of DESIGN.md §2) on
the same generated graph the GPU tests build.  Nothing here reads the CUDA path.

    python scripts/make_goldens.py rmat24:higher_id rmat24:lower_id rmat27:higher_id ...

Each file holds n, m, num_colors, rounds, the |W_r| trace, the SHA-256 of the colour array
(uint32 little-endian, vertex order), colours at 4096 seeded sample vertices (for locating a
mismatch), and the oracle's wall time on the machine that wrote it.
"""
import hashlib
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as wl  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def sample_ids(n: int, k: int = 4096, seed: int = 12345):
    """Seeded sample of vertex ids (SplitMix64 counter), shared with the GPU tests."""
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    return np.array([wl.splitmix64(seed + i) % n for i in range(min(k, n))], dtype=np.int64)


def colour_hash(c) -> str:
    return hashlib.sha256(np.ascontiguousarray(c, dtype="<u4").tobytes()).hexdigest()


def make(cfg: str, policy: str):
    t0 = time.time()
    g = wl.config_graph(cfg)
    tg = time.time() - t0
    t0 = time.perf_counter()
    c, nc, rd, tr = oracle.sgr(g, policy, trace=True)
    dt = time.perf_counter() - t0
    rc, bad = oracle.verify(g, c)
    assert rc == 0, (cfg, policy, rc, bad)
    ids = sample_ids(g.n)
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                            text=True).stdout.strip()
    out = {
        "config": cfg, "policy": policy, "n": g.n, "m": g.m, "max_degree": g.max_degree(),
        "num_colors": nc, "rounds": rd, "trace": tr,
        "sha256_colors_u32le": colour_hash(c),
        "sample_seed": 12345, "sample_ids": ids.tolist(), "sample_colors": c[ids].astype(int).tolist(),
        "oracle_seconds": round(dt, 2), "generate_seconds": round(tg, 2),
        "host": f"{platform.node()} {platform.processor() or platform.machine()}, 1 thread",
        "written_by": "scripts/make_goldens.py (oracle/ only)", "commit": commit,
    }
    path = os.path.join(GOLDEN, f"oracle_{cfg}_{policy}.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"{cfg} {policy}: n={g.n} m={g.m} colors={nc} rounds={rd} oracle {dt:.1f} s -> {path}", flush=True)


def main():
    for spec in sys.argv[1:]:
        cfg, policy = spec.split(":")
        make(cfg, policy)


if __name__ == "__main__":
    main()
