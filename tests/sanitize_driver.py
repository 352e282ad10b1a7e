"""Small colourings through the C ABI for compute-sanitizer (tests/test_sanitizer.py runs this
file under memcheck / racecheck / synccheck / initcheck).  Not a pytest module."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1606_06025_b200 as gc  # noqa: E402
import workloads as wl  # noqa: E402

graphs = [wl.rmat(10, 8, seed=3), wl.stencil27(6, 5, 4), wl.complete(130), wl.star(2000, center_last=True),
          wl.mesh2d(30, 20, 0.3)]
for g in graphs:
    rp = torch.from_numpy(g.row_ptr).cuda()
    ci = torch.from_numpy(g.col_idx).cuda()
    for pol in ("higher_id", "lower_id", "degree"):
        for kw in (dict(), dict(tuning=dict(n1=2, dense_div=1)), dict(warp_bin_max=8), dict(host_rounds=True)):
            if kw.get("host_rounds") and pol != "higher_id":
                continue
            res = gc.color(rp, ci, policy=pol, trace=True, **kw)
            ref, nc, r = oracle.sgr(g, pol)
            assert np.array_equal(res.colors.cpu().numpy().view(np.uint32), ref), (g.name, pol, kw)
        assert gc.verify(rp, ci, res.colors) == -1
print("sanitize_driver ok")
