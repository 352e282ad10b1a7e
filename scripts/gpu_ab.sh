set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for lib in ${LIBS:-default}; do
  for c in ${CONFIGS:-rmat24 stencil128 mesh8192}; do
    if [ "$lib" = default ]; then unset GC_LIB_PATH; else export GC_LIB_PATH=$PWD/$lib; fi
    echo "== $lib $c"; timeout 600 python scripts/perf.py --config $c --sweep ${SWEEP:-default} 2>&1 | tail -8
  done
done
