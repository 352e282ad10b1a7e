export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python scripts/perf.py --config rmat24 --sweep bins
for c in mesh8192 stencil128; do timeout 600 python scripts/perf.py --config $c 2>&1 | tail -1; done
