"""Sustained self-attention (5 entries x 13 visible blocks, Wan-1.3B shape)
with nvidia-smi sampling: SM clock, power and throttle reasons under load,
and TFLOP/s per MHz (the clock-independent figure to compare variants by).
usage: python scripts/attn_power.py [lib.so ...]"""
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2511_20426_b200 import _native as N  # noqa: E402


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        try:
            mhz, watts, reasons = [x.strip() for x in r.stdout.strip().split(",")]
            out.append((float(mhz), float(watts), reasons))
        except ValueError:
            pass
        time.sleep(0.1)


def run(lib, seconds=4.0, n_ent=5, n_vis=13, T=4680, heads=12):
    N.LIB_PATH = lib
    N._lib = None
    arena = torch.randn(13, 2, T, heads * 128, device="cuda").bfloat16()
    q = torch.randn(n_ent * T, heads * 128, device="cuda").bfloat16()
    out = torch.empty_like(q)
    b = N.make_batch(3, list(range(n_ent)), [0.0] * n_ent, [0] * n_ent, [list(range(n_vis))] * n_ent)
    mat = T * heads * 128
    f = lambda: N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(arena), N.ptr(arena) + mat * 2, 2 * mat, T, b,
                                                   T, heads, N.ptr(out), N.stream_ptr()), "attn")
    f()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, samples))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(20):
        f()
    th.start()
    s.record()
    n = 0
    t0 = time.time()
    while time.time() - t0 < seconds:
        for _ in range(10):
            f()
        n += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / n
    tf = 4.0 * n_ent * T * (n_vis * T) * heads * 128 / ms / 1e9
    load = samples[2:] if len(samples) > 4 else samples
    mhz = sorted(x[0] for x in load)[len(load) // 2]
    watts = sorted(x[1] for x in load)[len(load) // 2]
    reasons = sorted(set(x[2] for x in load))
    print(f"{lib}: {ms:.3f} ms {tf:.0f} TFLOP/s  sm {mhz:.0f} MHz  {watts:.0f} W  reasons {reasons}  "
          f"-> {tf / mhz * 1000:.1f} GFLOP/s per MHz ({100 * tf / (148 * 8192 * mhz * 1e6 / 1e12):.1f}% of the "
          f"tensor peak at that clock)")


if __name__ == "__main__":
    libs = sys.argv[1:] or [N.LIB_PATH]
    for lib in libs:
        run(lib, T=int(os.environ.get("BC_POWER_T", "4680")))
