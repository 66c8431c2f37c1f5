import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2511_20426_b200 import _native as N
M, Nn, K = 23400, 1536, 1536
A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(Nn, K, device="cuda").bfloat16()
C = torch.zeros(M, Nn, device="cuda"); gate = torch.ones(1, Nn, device="cuda")
for _ in range(5):
    N.check(N.lib().bc_gemm_bf16(N.ptr(A), N.ptr(B), N.ptr(C), M, Nn, K, 3, 0, N.ptr(gate), Nn, M, N.stream_ptr()), "g")
torch.cuda.synchronize()
