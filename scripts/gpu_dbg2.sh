export PYTHONUNBUFFERED=1
for lib in libgc_plain.so libgc_cgq.so libgc.so; do
echo "== $lib"
export GC_LIB_PATH=$PWD/paper_1606_06025_b200/csrc/$lib
for s in 11 12 13 14 15 16 13 14; do timeout 60 python scripts/dbg.py $s "dict(host_rounds=True)" 2>&1 | tail -1 | cut -c1-60; done
for c in rmat24 mesh8192; do timeout 600 python scripts/perf.py --config $c 2>&1 | tail -1; done
done
