export PYTHONUNBUFFERED=1
for c in rmat24 mesh8192 stencil128; do timeout 600 python scripts/perf.py --config $c 2>&1 | tail -1; done
