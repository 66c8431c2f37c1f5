"""Same-shape comparison of the self-attention kernel with the library
attention available on the box (NOT reference code; context for the
roofline fraction): torch SDPA (cuDNN / flash backends) and flashinfer's
prefill, on the steady-state cascade shape (5 entries x 4680 queries, 13
visible blocks = 60,840 keys, 12 heads x 128, bf16, non-causal)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_20426_b200 import _native as N

T, heads, n_ent, n_vis = 4680, 12, 5, 13
Nk = n_vis * T
flops = 4.0 * n_ent * T * Nk * heads * 128


def timeit(f, iters=5):
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


arena = torch.randn(n_vis, 2, T, heads * 128, device="cuda").bfloat16()
q = torch.randn(n_ent * T, heads * 128, device="cuda").bfloat16()
out = torch.empty_like(q)
b = N.make_batch(3, list(range(n_ent)), [0.0] * n_ent, [0] * n_ent, [list(range(n_vis))] * n_ent)
mat = T * heads * 128
ours = timeit(lambda: N.check(N.lib().bc_attention_paged(
    N.ptr(q), N.ptr(arena), N.ptr(arena) + mat * 2, 2 * mat, T, b, T, heads, N.ptr(out), N.stream_ptr()), "a"))
print(f"ours (paged slots)        {ours:8.3f} ms  {flops / ours / 1e9:7.0f} TFLOP/s")

# dense layouts for the libraries: K/V of all visible blocks concatenated
k = arena[:, 0].reshape(Nk, heads, 128)
v = arena[:, 1].reshape(Nk, heads, 128)
qd = q.view(n_ent, T, heads, 128).transpose(1, 2)               # [B, H, T, D]
kd = k.transpose(0, 1).unsqueeze(0).expand(n_ent, -1, -1, -1)   # [B, H, Nk, D]
vd = v.transpose(0, 1).unsqueeze(0).expand(n_ent, -1, -1, -1)
from torch.nn.attention import SDPBackend, sdpa_kernel
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel(be):
            ms = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qd, kd, vd))
        print(f"torch sdpa {name:14s} {ms:8.3f} ms  {flops / ms / 1e9:7.0f} TFLOP/s")
    except Exception as ex:  # backend unavailable for this shape / build
        print(f"torch sdpa {name:14s} unavailable ({type(ex).__name__}: {str(ex)[:80]})")
try:
    import flashinfer
    qf = q.view(n_ent, T, heads, 128)
    ms = timeit(lambda: [flashinfer.single_prefill_with_kv_cache(qf[e], k, v, causal=False)
                         for e in range(n_ent)])
    print(f"flashinfer single_prefill {ms:8.3f} ms  {flops / ms / 1e9:7.0f} TFLOP/s")
except Exception as ex:
    print(f"flashinfer unavailable ({type(ex).__name__}: {str(ex)[:120]})")
# flashinfer's Blackwell kernels on the same shape: the CUTLASS sm100 FMHA
# (fmha_varlen, JIT-built from flashinfer's bundled CUTLASS) over per-entry
# KV segments, and the trtllm-gen paged context kernel (prebuilt cubins; on an
# offline box it reports unavailable)
qf = q.view(n_ent * T, heads, 128)
try:
    from flashinfer.prefill import fmha_varlen
    kr = k.repeat(n_ent, 1, 1).contiguous()
    vr = v.repeat(n_ent, 1, 1).contiguous()
    qo = torch.arange(0, n_ent + 1, device="cuda", dtype=torch.int32) * T
    kvo = torch.arange(0, n_ent + 1, device="cuda", dtype=torch.int32) * Nk
    ms = timeit(lambda: fmha_varlen(qf, kr, vr, qo, kvo, max_qo_len=T, causal=False))
    print(f"flashinfer cutlass sm100 fmha {ms:8.3f} ms  {flops / ms / 1e9:7.0f} TFLOP/s")
    del kr, vr
except Exception as ex:
    print(f"flashinfer cutlass sm100 fmha unavailable ({type(ex).__name__}: {str(ex)[:160]})")
try:
    from flashinfer.prefill import trtllm_batch_context_with_kv_cache
    page = 32
    n_pages = (Nk + page - 1) // page
    kc = torch.zeros(n_pages * page, heads, 128, device="cuda", dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    kc[:Nk] = k
    vc[:Nk] = v
    kc = kc.view(n_pages, page, heads, 128).transpose(1, 2).contiguous()  # HND pages
    vc = vc.view(n_pages, page, heads, 128).transpose(1, 2).contiguous()
    tables = torch.arange(n_pages, device="cuda", dtype=torch.int32).unsqueeze(0).repeat(n_ent, 1)
    seq = torch.full((n_ent,), Nk, device="cuda", dtype=torch.int32)
    cq = torch.arange(0, n_ent + 1, device="cuda", dtype=torch.int32) * T
    ckv = torch.arange(0, n_ent + 1, device="cuda", dtype=torch.int32) * Nk
    ws = torch.zeros(256 << 20, device="cuda", dtype=torch.uint8)
    ms = timeit(lambda: trtllm_batch_context_with_kv_cache(qf, (kc, vc), ws, tables, seq, T, Nk, 128 ** -0.5, 1.0,
                                                           n_ent, cq, ckv, causal=False))
    print(f"flashinfer trtllm-gen context {ms:8.3f} ms  {flops / ms / 1e9:7.0f} TFLOP/s")
except Exception as ex:
    print(f"flashinfer trtllm-gen context unavailable ({type(ex).__name__}: {str(ex)[:160]})")
