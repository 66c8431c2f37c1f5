import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2511_20426_b200 import _native as N
def run(M, Nn, K, mode, bn=0, iters=20, cg=0):
    A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(Nn, K, device="cuda").bfloat16()
    C = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16 if mode in (0,1) else torch.float32)
    f = lambda: N.check(N.lib().bc_gemm_bf16(N.ptr(A), N.ptr(B), N.ptr(C), M, Nn, K, mode | ((bn//64)<<8) | (cg<<16), 0, 0, 0, 1, N.stream_ptr()), "g")
    for _ in range(3): f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    # torch reference
    for _ in range(3): torch.matmul(A, B.T)
    s.record()
    for _ in range(iters): torch.matmul(A, B.T)
    e.record(); torch.cuda.synchronize(); tms = s.elapsed_time(e)/iters
    fl = 2.0*M*Nn*K
    print(f"M={M} N={Nn} K={K} mode={mode} bn={bn} cg={cg}: {ms*1e3:.1f} us {fl/ms/1e9:.0f} TFLOP/s | cublas {tms*1e3:.1f} us {fl/tms/1e9:.0f} TFLOP/s")
for (M,Nn,K) in [(4680,4608,1536),(4680,1536,1536),(4680,8960,1536),(4680,1536,8960),(23400,4608,1536),(23400,8960,1536),(23400,1536,8960),(8192,8192,8192)]:
    for bn, cg in ((256, 1), (256, 2)):
        run(M,Nn,K,0,bn,cg=cg)
for (M,Nn,K) in [(23400,1536,1536),(23400,1536,8960),(4680,1536,1536)]:
    for bn, cg in ((256, 1), (256, 2)):
        run(M,Nn,K,3,bn,cg=cg)
