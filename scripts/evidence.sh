#!/bin/bash
# One GPU call that regenerates the round's evidence under gpurun_out/:
# GPU tests, the bench lines (1.3B default, 14B, LongLive-style), the
# steady-state launch list with DRAM bytes, ncu full captures of the
# dominant kernels, and the three sanitizers.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/ev_tests.txt
timeout 900 python bench.py 2>gpurun_out/ev_bench.err | tail -1 > gpurun_out/ev_bench.json
timeout 600 python scripts/wan_parity_report.py > gpurun_out/ev_parity.json 2>>gpurun_out/ev_bench.err
timeout 600 python scripts/attn_compare.py 2>/dev/null | grep -v Warn > gpurun_out/ev_attn_compare.txt
timeout 600 python scripts/attn_cross_bench.py 2>/dev/null | grep -v -i warn > gpurun_out/ev_attn_cross_compare.txt
timeout 900 python bench.py --preset 14b --steps 2 --no-cpu --no-switch 2>>gpurun_out/ev_bench.err | tail -1 > gpurun_out/ev_bench_14b.json
timeout 900 python bench.py --blocks 80 --sink 0 --switch-every 20 --steps 2 --no-cpu --no-seq --no-switch 2>>gpurun_out/ev_bench.err | tail -1 > gpurun_out/ev_bench_longlive.json
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/ev_launches.csv python scripts/profile_iter.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:attn -s 1 -c 1 -o gpurun_out/ev_attn python scripts/attn_one.py > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on -k regex:gemm_kernel -s 5 -c 2 -o gpurun_out/ev_gemm_ffn python scripts/profile_iter.py > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --set full -k regex:"ln_rows|qk_norm|rms_rows" -s 3 -c 3 -o gpurun_out/ev_bw python scripts/profile_iter.py > /dev/null 2>&1
timeout 900 python scripts/scaling_projection.py 2>/dev/null | tail -1 > gpurun_out/ev_scaling.json
BC_FORCE_DEVICE=0 BC_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --decode-gpu --steps 1 --warmup 1 \
  2>>gpurun_out/ev_bench.err | tail -1 > gpurun_out/ev_decode_gpu_one_gpu.json
timeout 300 python scripts/attn_power.py > gpurun_out/ev_attn_power.txt 2>&1
timeout 300 python scripts/gemm_tiling.py > gpurun_out/ev_gemm_tiling.txt 2>&1
# (compute-sanitizer may be closed on the pool; the loop then records that)
for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py 2>&1 | tail -4
done > gpurun_out/ev_sanitizers.txt
ls -la gpurun_out
