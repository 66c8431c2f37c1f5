import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_20426_b200 import _native as N
M, Nn, K = 23400, 4608, 1536
cg = int(os.environ.get("CG", "2"))
A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(Nn, K, device="cuda").bfloat16()
C = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    N.check(N.lib().bc_gemm_bf16(N.ptr(A), N.ptr(B), N.ptr(C), M, Nn, K, 0 | (4 << 8) | (cg << 16), 0, 0, 0, 1, N.stream_ptr()), "g")
torch.cuda.synchronize()
