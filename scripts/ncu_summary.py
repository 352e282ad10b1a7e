#!/usr/bin/env python
"""Summarise an ncu report: headline metrics + top stall SASS lines (run where ncu is)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
        "dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
        "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_read.sum",
        "lts__t_sectors_op_write.sum"]
def find(w):
    """Column of metric w: exact name, else a prefixed variant, else the .ratio
    form of a .pct metric (smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio)."""
    cands = [w] + ([w[:-4] + ".ratio"] if w.endswith(".pct") else [])
    for c in cands:
        if c in hdr:
            return hdr.index(c), c
        for i, h in enumerate(hdr):
            if h.endswith("." + c) or h.endswith(c):
                return i, h
    return None, None


for w in want:
    i, name = find(w)
    if i is None:
        print(f"{w:65s} {'(not reported)':>20s}")
    else:
        print(f"{name:65s} {vals[i]:>20s} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)"); i_e = h.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data) or 1
print(f"--- top {top} stall lines of {len(data)} SASS instructions")
for k, r in sorted(enumerate(data), key=lambda kr: -float(kr[1][i_s] or 0))[:top]:
    print(f"{float(r[i_s])/tot*100:5.1f}% #{k:5d} {r[1][:64]:66s} exec={r[i_e]}")
