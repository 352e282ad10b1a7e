#!/usr/bin/env python
"""Per-CUDA-source-line stall samples of an ncu report (cuda,sass view): top lines."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []; fname = ""; hdr = None; tot = 0
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_e = hdr.index("Instructions Executed"); continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try: smp = float(r[i_s] or 0)
        except ValueError: continue
        tot += smp
        res.append((smp, fname, r[0], r[1][:90], r[i_e]))
tot = tot or 1
for smp, f, ln, src, ex in sorted(res, reverse=True)[:top]:
    print(f"{smp/tot*100:5.1f}% {f}:{ln:5s} exec={ex:>11s}  {src}")
