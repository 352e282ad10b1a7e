set -u
mkdir -p gpurun_out
for c in ${NCU_CONFIGS:-rmat24}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgr_persistent -s 1 -c 1 -o gpurun_out/prof_$c -f python scripts/perf.py --config $c --reps 1 > gpurun_out/ncu_$c.log 2>&1; echo ncu $c rc=$?
done
