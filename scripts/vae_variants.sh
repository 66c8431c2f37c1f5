#!/bin/bash
# Build VAE-conv variants (compile-time switches) into /tmp and run the conv
# probe with each: usage scripts/vae_variants.sh "NAME:-DFLAG=.." ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cd "$ROOT/paper_2511_20426_b200/csrc"
NV="nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
NPR=$(python -c "import numpy,os;print(os.path.join(os.path.dirname(numpy.__file__),'random','lib'))")
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  OUT=/tmp/bcvae_$name; mkdir -p $OUT
  for f in *.cu; do $NV $flags -c $f -o $OUT/${f%.cu}.o & done; wait
  for f in *.cpp; do g++ -O3 -std=c++17 -fPIC -c $f -o $OUT/${f%.cpp}.o; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libbcb200.so $OUT/*.o -L$NPR -lnpyrandom -lm -lpthread
done
cd "$ROOT"
for spec in "$@"; do
  name=${spec%%:*}
  echo "== $name"
  python - <<PY
import sys; sys.path.insert(0, "$ROOT")
from paper_2511_20426_b200 import _native as N
N.LIB_PATH = "/tmp/bcvae_$name/libbcb200.so"
sys.argv = ["x"]
exec(open("$ROOT/scripts/vae_conv_probe.py").read())
PY
done
