import torch
X = torch.randn(23400, 1536, device="cuda")
def t(f, n=20):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / n * 1e3
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
def cold(f):
    def g():
        flush.zero_(); f()
    return g
conv = lambda: X.to(torch.bfloat16)
ln = lambda: torch.nn.functional.layer_norm(X, (1536,)).to(torch.bfloat16)
print("convert fp32->bf16 warm  %.1f us" % t(conv))
print("flush only              %.1f us" % t(flush.zero_))
print("flush + convert         %.1f us" % t(cold(conv)))
print("flush + torch LN+convert %.1f us" % t(cold(ln)))
print("copy fp32 (216 MB r+w)  %.1f us" % t(lambda: X.clone()))
