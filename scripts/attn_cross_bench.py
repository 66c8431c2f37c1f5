"""Text cross-attention shape through the paged API (5 entries x 4680 query
rows, ONE 512-token K/V 'slot' shared by every entry, 12 heads): ms per
launch and TFLOP/s, best of 5 rounds of 20 launches."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2511_20426_b200 import _native as N  # noqa: E402

n_ent, T, Tk, heads = 5, 4680, 512, 12
kv = torch.randn(1, 2, Tk, heads * 128, device="cuda").bfloat16()
q = torch.randn(n_ent * T, heads * 128, device="cuda").bfloat16()
out = torch.empty_like(q)
b = N.make_batch(3, list(range(n_ent)), [0.0] * n_ent, [0] * n_ent, [[0]] * n_ent)
mat = Tk * heads * 128
f = lambda: N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(kv), N.ptr(kv) + mat * 2, 2 * mat, Tk, b, T, heads,
                                               N.ptr(out), N.stream_ptr()), "attn")
for _ in range(5):
    f()
best = 1e9
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 20)
fl = 4.0 * n_ent * T * Tk * heads * 128
print(f"cross-attention shape: {best * 1e3:.1f} us  {fl / best / 1e9:.0f} TFLOP/s")


def timeit(g):
    for _ in range(3):
        g()
    b2 = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            g()
        e.record()
        torch.cuda.synchronize()
        b2 = min(b2, s.elapsed_time(e) / 20)
    return b2


# the libraries on the same shape (context for the fraction of peak)
k = kv[0, 0].view(Tk, heads, 128)
v = kv[0, 1].view(Tk, heads, 128)
qd = q.view(n_ent, T, heads, 128).transpose(1, 2)
kd = k.transpose(0, 1).unsqueeze(0).expand(n_ent, -1, -1, -1)
vd = v.transpose(0, 1).unsqueeze(0).expand(n_ent, -1, -1, -1)
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402
try:
    with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
        ms = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qd, kd, vd))
    print(f"torch sdpa cudnn: {ms * 1e3:.1f} us  {fl / ms / 1e9:.0f} TFLOP/s")
except Exception as ex:
    print(f"torch sdpa cudnn unavailable ({type(ex).__name__})")
qf = q.view(n_ent * T, heads, 128)
try:
    from flashinfer.prefill import trtllm_batch_context_with_kv_cache
    page = 32
    n_pages = Tk // page
    kc = k.view(n_pages, page, heads, 128).transpose(1, 2).contiguous()
    vc = v.view(n_pages, page, heads, 128).transpose(1, 2).contiguous()
    tables = torch.arange(n_pages, device="cuda", dtype=torch.int32).unsqueeze(0).repeat(n_ent, 1)
    seq = torch.full((n_ent,), Tk, device="cuda", dtype=torch.int32)
    cq = torch.arange(0, n_ent + 1, device="cuda", dtype=torch.int32) * T
    ckv = torch.arange(0, n_ent + 1, device="cuda", dtype=torch.int32) * Tk
    ws = torch.zeros(256 << 20, device="cuda", dtype=torch.uint8)
    ms = timeit(lambda: trtllm_batch_context_with_kv_cache(qf, (kc, vc), ws, tables, seq, T, Tk, 128 ** -0.5, 1.0,
                                                           n_ent, cq, ckv, causal=False))
    print(f"flashinfer trtllm-gen context: {ms * 1e3:.1f} us  {fl / ms / 1e9:.0f} TFLOP/s")
except Exception as ex:
    print(f"flashinfer trtllm-gen unavailable ({type(ex).__name__}: {str(ex)[:120]})")
try:
    from flashinfer.prefill import fmha_varlen
    kr = k.repeat(n_ent, 1, 1).contiguous()
    vr = v.repeat(n_ent, 1, 1).contiguous()
    qo = torch.arange(0, n_ent + 1, device="cuda", dtype=torch.int32) * T
    kvo = torch.arange(0, n_ent + 1, device="cuda", dtype=torch.int32) * Tk
    ms = timeit(lambda: fmha_varlen(qf, kr, vr, qo, kvo, max_qo_len=T, causal=False))
    print(f"flashinfer cutlass sm100 fmha: {ms * 1e3:.1f} us  {fl / ms / 1e9:.0f} TFLOP/s")
except Exception as ex:
    print(f"flashinfer cutlass sm100 fmha unavailable ({type(ex).__name__}: {str(ex)[:120]})")
