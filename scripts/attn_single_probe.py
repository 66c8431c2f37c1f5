import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2511_20426_b200 import _native as N
T, heads, n_vis = 4680, 12, 13
for qn, n_ent in ((128, 12), (256, 12)):
    arena = torch.randn(n_vis, 2, T, heads * 128, device="cuda").bfloat16()
    q = torch.randn(n_ent * qn, heads * 128, device="cuda").bfloat16()
    out = torch.empty_like(q)
    b = N.make_batch(3, list(range(n_ent)), [0.0] * n_ent, [0] * n_ent, [list(range(n_vis))] * n_ent)
    mat = T * heads * 128
    f = lambda: N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(arena), N.ptr(arena) + mat * 2, 2 * mat, T, b, qn, heads, N.ptr(out), N.stream_ptr()), "a")
    for _ in range(3): f()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        s.record()
        for _ in range(10): f()
        e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e) / 10)
    print(f"q rows/entry {qn} x {n_ent} entries x {heads} heads (single-tile items: {qn == 128}): {best*1e3:.1f} us")
