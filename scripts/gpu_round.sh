set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
for c in rmat24 stencil128 mesh8192; do timeout 600 python scripts/perf.py --config $c --sweep ${SWEEP:-default} > gpurun_out/perf_$c.log 2>&1; cat gpurun_out/perf_$c.log; done
for c in rmat24 mesh8192; do GC_L2_PERSIST=0 timeout 600 python scripts/perf.py --config $c  > gpurun_out/perf_persist_$c.log 2>&1; echo persist; cat gpurun_out/perf_persist_$c.log; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgr_persistent -s 1 -c 1 -o gpurun_out/prof_rmat24 python scripts/perf.py --config rmat24 --reps 1 > gpurun_out/ncu_rmat24.log 2>&1; echo ncu rc=$?
