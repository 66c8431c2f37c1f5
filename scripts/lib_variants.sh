#!/bin/bash
# Build library variants (compile-time -D switches) into OUTROOT (default
# build/variants, shipped to the GPU box with the tree) and run a script
# against each: scripts/lib_variants.sh build "NAME:-DFLAG=.." ...
#              scripts/lib_variants.sh run script.py NAME ...
# (the script sees BC_LIB=<variant .so>; _native honours it)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUTROOT=${OUTROOT:-$ROOT/build/variants}
cmd=$1; shift
if [ "$cmd" = build ]; then
  cd "$ROOT/paper_2511_20426_b200/csrc"
  NV="nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -lineinfo"
  NPR=$(python -c "import numpy,os;print(os.path.join(os.path.dirname(numpy.__file__),'random','lib'))")
  for spec in "$@"; do
    name=${spec%%:*}; flags=${spec#*:}
    OUT=$OUTROOT/bcv_$name; mkdir -p $OUT
    for f in *.cu; do $NV $flags -c $f -o $OUT/${f%.cu}.o 2>$OUT/${f%.cu}.log & done; wait
    for f in *.cu; do  # a failed compile must not leave a .so with missing symbols
      [ -f $OUT/${f%.cu}.o ] || { echo "variant $name: $f failed"; cat $OUT/${f%.cu}.log; exit 1; }
    done
    rm -f $OUT/*.log
    for f in *.cpp; do g++ -O3 -std=c++17 -fPIC -c $f -o $OUT/${f%.cpp}.o; done
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libbcb200.so $OUT/*.o -L$NPR -lnpyrandom -lm -lpthread
    rm -f $OUT/*.o
  done
else
  script=$1; shift
  for name in "$@"; do
    echo "== $name"
    BC_LIB=$OUTROOT/bcv_$name/libbcb200.so python "$ROOT/$script"
  done
fi
