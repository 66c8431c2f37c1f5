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
