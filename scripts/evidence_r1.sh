#!/bin/bash
# One GPU call that regenerates the round's evidence under gpurun_out/:
# GPU tests, the default bench line, the steady-state launch list, ncu full
# captures of the dominant kernels, and the three sanitizers.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev_tests.txt
timeout 900 python bench.py 2>gpurun_out/ev_bench.err | tail -1 > gpurun_out/ev_bench.json
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ev_launches.csv python scripts/profile_iter.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:attn -s 1 -c 1 -o gpurun_out/ev_attn python scripts/attn_one.py > /dev/null 2>&1
CG=2 timeout 600 ncu --set full --import-source on -k regex:gemm -s 1 -c 1 -o gpurun_out/ev_gemm_pair python scripts/gemm_one.py > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py 2>&1 | tail -4
done > gpurun_out/ev_sanitizers.txt
ls -la gpurun_out
