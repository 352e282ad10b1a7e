# Bench lines + ncu evidence on the GPU box (run through gpurun from the repo root).
#   COMMIT=<sha> CONFIGS="rmat24 stencil128 mesh8192" NCU_CONFIGS="rmat24" bash scripts/gpu_bench.sh
set -u
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for c in ${CONFIGS:-rmat24}; do
  extra=""; [ "$c" != rmat24 ] && extra="--no-cpu"
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 $extra > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log | cut -c1-400
done
if [ -n "${REFERENCE:-}" ]; then
  timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1; tail -1 gpurun_out/bench_reference.log | cut -c1-300
fi
if [ -n "${LAUNCHES:-1}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat24.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu launches rc=$?
fi
for c in ${NCU_CONFIGS:-rmat24}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgr_persistent -s 2 -c 1 -o gpurun_out/prof_$c -f python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_$c.log 2>&1; echo ncu full $c rc=$?
  (python scripts/ncu_summary.py gpurun_out/prof_$c.ncu-rep 30; echo "--- top 30 CUDA source lines (stall samples)"; python scripts/ncu_lines.py gpurun_out/prof_$c.ncu-rep 30) > gpurun_out/summary_$c.txt 2>&1
  ncu -i gpurun_out/prof_$c.ncu-rep --page raw --csv > gpurun_out/raw_$c.csv 2>/dev/null
  python scripts/ncu_record.py $c gpurun_out/raw_$c.csv --commit ${COMMIT:-unknown} > gpurun_out/ncu_record_$c.log 2>&1
  if [ "$c" != "${KEEP_REP:-rmat24}" ]; then rm -f gpurun_out/prof_$c.ncu-rep; fi
done
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
du -sh gpurun_out
