"""The gated-residual GEMMs of a cascade iteration (o / co projections at the
width-5 batch, the width-1 sequential rows, a G=8 slice) and FFN2, auto
tiling, best of 3 rounds of 30 launches."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2511_20426_b200 import _native as N  # noqa: E402


def bench(M, Nn, K, iters=30):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(Nn, K, device="cuda").bfloat16()
    C = torch.zeros(M, Nn, device="cuda")
    gate = torch.ones(1, Nn, device="cuda")
    f = lambda: N.check(N.lib().bc_gemm_bf16(N.ptr(A), N.ptr(B), N.ptr(C), M, Nn, K, 3, 0, N.ptr(gate), Nn, M,
                                             N.stream_ptr()), "gemm")
    for _ in range(3):
        f()
    best = 1e9
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            f()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / iters * 1e3)
    print(f"M={M:5d} N={Nn} K={K}: {best:7.1f} us  {2.0 * M * Nn * K / best / 1e6:6.0f} TFLOP/s  "
          f"{8.0 * M * Nn / best / 1e3:6.0f} GB/s residual")


for M, Nn, K in [(23400, 1536, 1536), (4680, 1536, 1536), (2925, 1536, 1536), (23400, 1536, 8960)]:
    bench(M, Nn, K)
