"""Every tiling of the tcgen05 GEMM on the DiT's shapes at small and large M
(width-1 sequential rows, the G=8 row slice, the width-5 cascade batch),
back to back so that clock drift hits all tilings alike; the automatic
choice (gemm_plan) is printed beside the fastest.  The epilogue mode is the
one the shape runs with in the step (3 = gated fp32 residual for N = 1536).
usage: python scripts/gemm_tiling.py"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2511_20426_b200 import _native as N  # noqa: E402

TILINGS = [(256, 2), (224, 2), (192, 2), (256, 1), (128, 1)]


def bench(M, Nn, K, mode, bn, cg, A, B, C, gate, iters=30):
    f = lambda: N.check(N.lib().bc_gemm_bf16(N.ptr(A), N.ptr(B), N.ptr(C), M, Nn, K,
                                             mode | (((bn // 64) << 8) if bn % 64 == 0 else ((bn // 32) << 8) | (1 << 18)) | (cg << 16), 0,
                                             N.ptr(gate) if gate is not None else 0, Nn if gate is not None else 0,
                                             M, N.stream_ptr()), "gemm")
    for _ in range(3):
        f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    shapes = []
    for M in (4680, 2925, 23400):
        shapes += [(M, 4608, 1536, 0), (M, 1536, 1536, 3), (M, 8960, 1536, 1), (M, 1536, 8960, 3)]
    for M, Nn, K, mode in shapes:
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = torch.randn(Nn, K, device="cuda").bfloat16()
        C = torch.zeros(M, Nn, device="cuda", dtype=torch.float32 if mode == 3 else torch.bfloat16)
        gate = torch.ones(1, Nn, device="cuda") if mode == 3 else None
        res = {}
        for bn, cg in TILINGS:
            if Nn % bn and bn != 224:
                continue
            res[(bn, cg)] = bench(M, Nn, K, mode, bn, cg, A, B, C, gate)
        auto = bench(M, Nn, K, mode, 0, 0, A, B, C, gate)
        best = min(res, key=res.get)
        fl = 2.0 * M * Nn * K
        cells = "  ".join(f"{bn}x{cg}:{us:7.1f}" for (bn, cg), us in res.items())
        print(f"M={M:5d} N={Nn:4d} K={K:4d} mode={mode}  {cells}  | auto {auto:7.1f} us "
              f"({fl / auto / 1e6:.0f} TFLOP/s)  best {best[0]}x{best[1]} {res[best]:.1f} us")


if __name__ == "__main__":
    main()
