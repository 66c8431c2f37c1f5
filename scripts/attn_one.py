"""One steady-state-shaped attention launch (5 entries x 13 visible blocks,
Wan-1.3B head geometry) for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_20426_b200 import _native as N
T, heads, n_ent, n_vis = 4680, 12, 5, 13
arena = torch.randn(13, 2, T, heads * 128, device="cuda").bfloat16()
q = torch.randn(n_ent * T, heads * 128, device="cuda").bfloat16()
out = torch.empty_like(q)
b = N.make_batch(3, list(range(n_ent)), [0.0] * n_ent, [0] * n_ent, [list(range(n_vis))] * n_ent)
mat = T * heads * 128
for _ in range(int(os.environ.get("REPS", "2"))):
    N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(arena), N.ptr(arena) + mat * 2, 2 * mat, T, b, T,
                                       heads, N.ptr(out), N.stream_ptr()), "attn")
torch.cuda.synchronize()
