import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_06025_b200 as gc
for bps in (4, 0):
    print(os.environ.get("GC_LIB_PATH", "default"), "blocks/SM", bps, "us per grid barrier", round(gc.bench_grid_sync(0, bps, 4000), 3))
