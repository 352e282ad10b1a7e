import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1606_06025_b200 as gc, workloads as wl
cfg = sys.argv[1]
g = wl.config_graph(cfg)
rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
for n1 in sys.argv[2:]:
    os.environ["GC_N1"] = n1
    r = gc.color(rp, ci, validate=False, count_work=True)
    print(cfg, "N1=" + n1, json.dumps(r.work))
    r = gc.color(rp, ci, validate=False, phase_times=True)
    a = [x for x, y in r.phase_us]; b = [y for x, y in r.phase_us]
    print("  A total %.1f us, B total %.1f us; rounds %d" % (sum(a), sum(b), r.rounds))
    for i in list(range(0, min(12, r.rounds))) + list(range(40, r.rounds, 20)):
        print("   r=%3d A=%7.1f B=%7.1f |W|=%d" % (i + 1, a[i], b[i], r.trace[i]))
# (appended) kernel time vs phase sums: the remainder is ingest + finalize
if os.environ.get("KTIME"):
    r = gc.color(rp, ci, validate=False, time_kernel=True)
    r2 = gc.color(rp, ci, validate=False, phase_times=True)
    a = sum(x for x, y in r2.phase_us); b = sum(y for x, y in r2.phase_us)
    print("kernel %.1f us, A %.1f, B %.1f, ingest+finalize ~%.1f" % (r.kernel_ms * 1e3, a, b, r.kernel_ms * 1e3 - a - b))
