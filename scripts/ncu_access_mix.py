#!/usr/bin/env python
"""Memory-access mix of one kernel launch from an ncu report (SASS view, each instruction once):
per opcode the warp instructions, thread accesses and L2 sectors requested, plus the time the
launch would need if every scattered access class ran at the rate measured alone by
scripts/probes/l2_ceiling.cu (gathers, REDs) — the "scattered-access ceiling" of DESIGN.md §7.

    python scripts/ncu_access_mix.py gpurun_out/prof_rmat24.ncu-rep [profiles/r02_l2_ceiling.jsonl]
"""
import collections
import csv
import io
import json
import subprocess
import sys


def access_mix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    hdr = None
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        toks = [t for t in d["Source"].replace(";", "").split() if not t.startswith("@")]
        if not toks or not toks[0].startswith(("LDG", "STG", "RED", "ATOM", "LDS", "STS")):
            continue
        try:
            ins = float(d["Instructions Executed"] or 0)
            th = float(d["Predicated-On Thread Instructions Executed"] or 0)
            sec = float(d["L2 Theoretical Sectors Global"] or 0)
        except ValueError:
            continue
        a = agg[toks[0]]
        a[0] += ins
        a[1] += th
        a[2] += sec
    return agg


def main():
    rep = sys.argv[1]
    ceil = {}
    if len(sys.argv) > 2:
        for line in open(sys.argv[2]):
            d = json.loads(line)
            if d["footprint_bytes"] < 20e6 and d["ctas_per_sm"] == 4:  # L2-resident, the kernel's grid
                ceil[d["kind"]] = d["gacc_per_s"] * 1e9
    agg = access_mix(rep)
    print("%-26s %12s %14s %14s" % ("opcode", "warp-inst", "thread-acc", "L2 sectors"))
    for k, (ins, th, sec) in sorted(agg.items(), key=lambda x: -x[1][2]):
        if ins:
            print("%-26s %12.4g %14.4g %14.4g" % (k, ins, th, sec))
    tot = sum(v[2] for v in agg.values())
    print("global L2 sectors requested: %.4g (%.1f GB)" % (tot, tot * 32 / 1e9))
    if ceil:
        g = agg.get("LDG.E.U8.STRONG.GPU", [0, 0, 0])[1]
        red = agg.get("REDG.E.OR.STRONG.GPU", [0, 0, 0])[1]
        tg = g / ceil["gather_idx"] * 1e3
        tr = red / ceil["red_idx"] * 1e3
        print("state-word gathers %.4g at %.0f G/s alone: %.2f ms; plane REDs %.4g at %.0f G/s alone: %.2f ms; "
              "sum %.2f ms" % (g, ceil["gather_idx"] / 1e9, tg, red, ceil["red_idx"] / 1e9, tr, tg + tr))


if __name__ == "__main__":
    main()
