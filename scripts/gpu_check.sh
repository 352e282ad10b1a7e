set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-rmat24 stencil128 mesh8192}; do for sw in ${SWEEPS:-default}; do timeout 600 python scripts/perf.py --config $c --sweep $sw > gpurun_out/perf_${c}_$sw.log 2>&1; head -c 2500 gpurun_out/perf_${c}_$sw.log; done; done
