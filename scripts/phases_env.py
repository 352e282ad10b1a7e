import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1606_06025_b200 as gc, workloads as wl
cfg = sys.argv[1]
g = wl.config_graph(cfg)
rp = torch.from_numpy(g.row_ptr).cuda(); ci = torch.from_numpy(g.col_idx).cuda()
for spec in sys.argv[2:]:
    env = dict(kv.split("=") for kv in spec.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    r = gc.color(rp, ci, validate=False, count_work=True)
    w = r.work
    r = gc.color(rp, ci, validate=False, phase_times=True)
    a = [x for x, y in r.phase_us]; b = [y for x, y in r.phase_us]
    print(cfg, spec, "A %.0f B %.0f us; evaluated %d marks %d" % (sum(a), sum(b), w["phase_b_evaluated"], w["dirty_marks"]))
    for i in [0, 1, 2, 3, 4, 5, 10, 20, 40, 60, 80, 100, 120, 140, 160, 180]:
        if i < r.rounds:
            print("   r=%3d A=%7.1f B=%7.1f |W|=%d" % (i + 1, a[i], b[i], r.trace[i]))
    for k, v in old.items():
        if v is None: os.environ.pop(k, None)
        else: os.environ[k] = v
