export PYTHONUNBUFFERED=1
for m in "dict(host_rounds=True)" "dict()" "dict(pull_firstfit=True)"; do
echo "== $m"
for s in 11 12 13 14 15 16 13 14 15 16; do timeout 60 python scripts/dbg.py $s "$m" 2>&1 | tail -1 | cut -c1-60; done
done
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
for c in rmat24 stencil128 mesh8192; do timeout 600 python scripts/perf.py --config $c > gpurun_out/perf_$c.log 2>&1; cat gpurun_out/perf_$c.log; done
