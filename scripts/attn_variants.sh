#!/bin/bash
# Build attention variants (compile-time switches) into /tmp and benchmark
# each: usage scripts/attn_variants.sh "NAME:-DFLAG=.. -DFLAG2=.." ...
# OUTROOT (default /tmp) holds the builds; SKIP_BUILD=1 only benchmarks
# (build here with OUTROOT=build/variants, run on the GPU box with SKIP_BUILD=1)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cd "$ROOT/paper_2511_20426_b200/csrc"
NV="nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
NPR=$(python -c "import numpy,os;print(os.path.join(os.path.dirname(numpy.__file__),'random','lib'))")
OUTROOT=${OUTROOT:-/tmp}
case "$OUTROOT" in /*) ;; *) OUTROOT="$ROOT/$OUTROOT";; esac
for spec in "$@"; do
  [ -n "$SKIP_BUILD" ] && break
  name=${spec%%:*}; flags=${spec#*:}
  OUT=$OUTROOT/bcv_$name; mkdir -p $OUT
  for f in *.cu; do $NV $flags -c $f -o $OUT/${f%.cu}.o & done; wait
  for f in *.cpp; do g++ -O3 -std=c++17 -fPIC -c $f -o $OUT/${f%.cpp}.o; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libbcb200.so $OUT/*.o -L$NPR -lnpyrandom -lm -lpthread
done
cd "$ROOT"
for spec in "$@"; do
  name=${spec%%:*}
  for poly in ${POLYS:-0}; do
    echo "== $name poly=$poly"
    BC_ATTN_POLY=$poly python - <<PY
import sys; sys.path.insert(0, "$ROOT")
from paper_2511_20426_b200 import _native as N
N.LIB_PATH = "$OUTROOT/bcv_$name/libbcb200.so"
exec(open("$ROOT/scripts/attn_bench.py").read().split("def run")[0])
exec("def run" + open("$ROOT/scripts/attn_bench.py").read().split("def run")[1])
PY
  done
done
