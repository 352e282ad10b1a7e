# A/B of library builds: bash scripts/ab.sh "default build/libgc_x.so ..." "rmat24 stencil128 mesh8192"
set -u
for c in $2; do
  for lib in $1; do
    if [ "$lib" = default ]; then unset GC_LIB_PATH; else export GC_LIB_PATH=$PWD/$lib; fi
    echo "$c $lib $(timeout 300 python scripts/perf.py --config $c --reps 9 2>&1 | tail -1 | cut -c1-160)"
  done
done
