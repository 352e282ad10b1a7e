set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for d in 4 0; do
GC_DENSE_DIV=$d timeout 300 compute-sanitizer --tool synccheck python scripts/dbg_case.py rmat13 "dict(thread_bin_max=1, warp_bin_max=2)" 2>&1 | head -12
done
GC_DENSE_DIV=4 timeout 300 compute-sanitizer --tool synccheck python scripts/dbg_case.py g500 "dict()" 2>&1 | head -12
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
