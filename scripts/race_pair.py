"""Racecheck target: one small CTA-pair GEMM per epilogue."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_20426_b200 import _native as N
A2 = torch.randn(600, 256, device="cuda").bfloat16(); B2 = torch.randn(512, 256, device="cuda").bfloat16()
for mode, dt in ((0, torch.bfloat16), (3, torch.float32)):
    C = torch.zeros(600, 512, device="cuda", dtype=dt)
    g = torch.ones(6, 512, device="cuda")
    N.check(N.lib().bc_gemm_bf16(N.ptr(A2), N.ptr(B2), N.ptr(C), 600, 512, 256, mode | (4 << 8) | (2 << 16), 0,
                                 N.ptr(g) if mode == 3 else 0, 512, 100, N.stream_ptr()), "gemm pair")
torch.cuda.synchronize()
print("done")
