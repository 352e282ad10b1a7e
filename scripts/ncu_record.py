#!/usr/bin/env python
"""Record the ncu numbers bench.py reports (roofline.traffic etc.) into profiles/ncu_traffic.json,
stamped with the commit that was profiled.

    python scripts/ncu_record.py <config> <raw.csv> [--commit C]

raw.csv = `ncu -i prof_<config>.ncu-rep --page raw --csv` of one `ncu --set full` launch of the
persistent kernel (scripts/gpu_ncu.sh).  Metric names are matched with or without this ncu's
section prefixes (e.g. FBSP.TriageCompute.dram__throughput...).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def col(hdr, name, vals=None):
    """Exact metric name first, else a section-prefixed variant that has a value."""
    if name in hdr:
        return hdr.index(name)
    for i, h in enumerate(hdr):
        if h.endswith("." + name) and (vals is None or vals[i]):
            return i
    return None


def main():
    cfg, path = sys.argv[1], sys.argv[2]
    commit = sys.argv[sys.argv.index("--commit") + 1] if "--commit" in sys.argv else subprocess.run(
        ["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"], capture_output=True, text=True).stdout.strip()
    rows = list(csv.reader(io.StringIO(open(path).read())))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name, scale=1.0):
        i = col(hdr, name, vals)
        if i is None or not vals[i]:
            return None
        v = float(vals[i].replace(",", ""))
        u = units[i]
        if u in ("Kbyte", "KB"):
            v *= 1e3
        elif u in ("Mbyte", "MB"):
            v *= 1e6
        elif u in ("Gbyte", "GB"):
            v *= 1e9
        elif u == "usecond":
            v *= 1e-3
        elif u == "nsecond":
            v *= 1e-6
        elif u == "msecond":
            pass
        return v * scale

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    rec = {
        "dram_bytes": (rd or 0) + (wr or 0), "dram_read_bytes": rd, "dram_write_bytes": wr,
        "kernel_ms": get("gpu__time_duration.sum"),
        "dram_throughput_pct": get("dram__throughput.avg.pct_of_peak_sustained_elapsed")
        or get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_hit_pct": get("lts__t_sector_hit_rate.pct"),
        "l2_throughput_pct": get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_sectors": get("lts__t_sectors.sum"),
        "global_ld_bytes_per_sector": get("smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio")
        or get("smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct"),
        "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": get("launch__registers_per_thread"),
        "source": f"ncu --set full --clock-control none, one launch of sgr_persistent (bench.py --config {cfg})",
    }
    out = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        allrec = json.load(open(out))
        if "configs" not in allrec:
            allrec = {"configs": {}}
    except Exception:
        allrec = {"configs": {}}
    allrec["configs"][cfg] = dict(rec, commit=commit)
    allrec["commit"] = commit
    with open(out, "w") as f:
        json.dump(allrec, f, indent=1)
    print(json.dumps({cfg: rec}))


if __name__ == "__main__":
    main()
