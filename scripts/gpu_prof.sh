set -u
mkdir -p gpurun_out
timeout 600 python bench.py --config rmat24 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_rmat24.log 2>&1; tail -1 gpurun_out/bench_rmat24.log
for c in ${CONFIGS:-rmat24}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgr_persistent -s 1 -c 1 -o gpurun_out/prof_$c python scripts/perf.py --config $c --reps 1 > gpurun_out/ncu_$c.log 2>&1; echo ncu $c rc=$?
done
