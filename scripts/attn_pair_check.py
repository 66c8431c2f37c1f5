"""Self-attention outputs for a few shapes, saved to an .npz (compare two
runs with different BC_ATTN_* settings: the CTA-pair kernel must equal the
single-CTA kernels bit for bit).  usage: python scripts/attn_pair_check.py OUT.npz"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_2511_20426_b200 import _native as N  # noqa: E402

out = {}
g = torch.Generator(device="cuda")
g.manual_seed(3)
for name, (n_ent, n_vis, T, heads) in {"a": (2, 3, 4680, 12), "b": (5, 13, 4680, 12), "c": (1, 2, 520, 2),
                                        "d": (3, 4, 1000, 4)}.items():
    arena = torch.randn(n_vis + 1, 2, T, heads * 128, device="cuda", generator=g).bfloat16()
    q = torch.randn(n_ent * T, heads * 128, device="cuda", generator=g).bfloat16()
    o = torch.zeros_like(q)
    vis = [list(range(n_vis - (i % 2))) for i in range(n_ent)]   # ragged visible lists
    b = N.make_batch(3, list(range(n_ent)), [0.0] * n_ent, [0] * n_ent, vis)
    mat = T * heads * 128
    N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(arena), N.ptr(arena) + mat * 2, 2 * mat, T, b, T, heads,
                                       N.ptr(o), N.stream_ptr()), "attn")
    torch.cuda.synchronize()
    out[name] = o.view(torch.int16).cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", {k: v.shape for k, v in out.items()})
