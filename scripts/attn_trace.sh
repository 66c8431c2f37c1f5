#!/bin/bash
# Build a tracing variant of the library (BC_ATTN_TRACE) into /tmp and dump
# the per-phase timeline of CTA (0,0,0) of a steady-state attention launch.
set -e
cd "$(dirname "$0")/../paper_2511_20426_b200/csrc"
# OUT (default /tmp/bc_trace): build dir; SKIP_BUILD=1 reuses it (build here
# into the repo tree, run on the GPU box); EXTRA: more -D flags
OUT=${OUT:-/tmp/bc_trace}
case "$OUT" in /*) ;; *) OUT="$(cd ../.. && pwd)/$OUT";; esac
mkdir -p $OUT
if [ -z "$SKIP_BUILD" ]; then
NV="nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
for f in *.cu; do $NV -DBC_ATTN_TRACE ${EXTRA:-} -c $f -o $OUT/${f%.cu}.o & done; wait
for f in *.cpp; do g++ -O3 -std=c++17 -fPIC -c $f -o $OUT/${f%.cpp}.o; done
NPR=$(python -c "import numpy,os;print(os.path.join(os.path.dirname(numpy.__file__),'random','lib'))")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libbcb200.so $OUT/*.o -L$NPR -lnpyrandom -lm -lpthread
rm -f $OUT/*.o
fi
cd ../..
export BC_TRACE_LIB=$OUT/libbcb200.so
python - <<'PY'
import ctypes, sys, numpy as np, os
sys.path.insert(0, os.getcwd())
from paper_2511_20426_b200 import _native as N
N.LIB_PATH = os.environ["BC_TRACE_LIB"]
import torch
T, heads, n_ent, n_vis = 4680, 12, 5, 13
Tk = T
if os.environ.get("CROSS"):  # the text cross-attention shape: one 512-token K/V slot
    Tk, n_vis = 512, 1
arena = torch.randn(n_vis, 2, Tk, heads * 128, device="cuda").bfloat16()
q = torch.randn(n_ent * T, heads * 128, device="cuda").bfloat16()
out = torch.empty_like(q)
b = N.make_batch(3, list(range(n_ent)), [0.0] * n_ent, [0] * n_ent, [list(range(n_vis))] * n_ent)
mat = Tk * heads * 128
for _ in range(3):
    N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(arena), N.ptr(arena) + mat * 2, 2 * mat, Tk, b, T,
                                       heads, N.ptr(out), N.stream_ptr()), "attn")
buf = (ctypes.c_ulonglong * (32 * 64 + 256 * 8))()
lib = ctypes.CDLL(N.LIB_PATH)
lib.bc_attn_trace_read(buf)
allbuf = np.array(buf, dtype=np.int64)
t = allbuf[:32 * 64].reshape(32, 64)
c = allbuf[32 * 64:].reshape(256, 8)
t0 = t[t > 0].min()
names = {0: "A s_full", 4: "A s_read", 1: "A max", 2: "A exp", 5: "A o_rdy", 3: "A p_full",
         8: "B s_full", 12: "B s_read", 9: "B max", 10: "B exp", 13: "B o_rdy", 11: "B p_full", 16: "M s_emptyA", 17: "M QK_A", 18: "M p_fullA", 19: "M PV_A", 20: "M s_emptyB",
         21: "M QK_B", 22: "M p_fullB", 23: "M PV_B", 24: "M K_rdy", 25: "M V_rdy"}
for j in (range(0, 8) if os.environ.get("CROSS") else range(20, 28)):
    row = {names[k]: int(t[k, j] - t0) for k in names if t[k, j] > 0}
    print(j, sorted(row.items(), key=lambda kv: kv[1]))
per = [int(t[1, j + 1] - t[1, j]) for j in range(20, 60) if t[1, j + 1] > 0 and t[1, j] > 0]
if per:
    print("A token period (cycles):", per, "median", int(np.median(per)))
c = c[c[:, 0] > 0]
if len(c):
    cyc, ns, tiles, wait, kv, se, iqk, ipv = c.T
    per = cyc / np.maximum(tiles, 1) * 2
    print(f"CTAs {len(c)}: cycles max {cyc.max()} mean {cyc.mean():.0f}; ns max {ns.max()}; clock {cyc.max() / ns.max():.3f} GHz")
    print(f"cycles per 2-tile key step: min {per.min():.0f} median {np.median(per):.0f} max {per.max():.0f}")
    print(f"issuer wait for P: {100 * wait.sum() / cyc.sum():.1f}% of cycles; for K/V: {100 * kv.sum() / cyc.sum():.1f}%")
    print(f"s_empty wait {100 * se.sum() / cyc.sum():.1f}%; QK issue {100 * iqk.sum() / cyc.sum():.1f}%; PV issue {100 * ipv.sum() / cyc.sum():.1f}%; tiles per CTA min {tiles.min()} max {tiles.max()}")
    busy = (tiles * 1024).sum() / (cyc.max() * len(c))
    print(f"tensor busy (1024 cyc per tile-key step) over the makespan: {100 * busy:.1f}%")
    print(f"per QK group issue {iqk.sum() / (tiles.sum()):.0f} cyc, per PV group {ipv.sum() / tiles.sum():.0f} cyc (8 MMAs = 512 cyc of pipe)")
PY
