export PYTHONUNBUFFERED=1
for k in 1 2 3; do for s in 12 13 14 15 16; do timeout 60 python scripts/dbg.py $s "dict()" 2>&1 | tail -1; done; done
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
for c in rmat24 stencil128 mesh8192; do timeout 600 python scripts/perf.py --config $c > gpurun_out/perf_$c.log 2>&1; cat gpurun_out/perf_$c.log; done
