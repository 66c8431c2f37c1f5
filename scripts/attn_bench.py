import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2511_20426_b200 import _native as N
def run(n_ent, n_vis, T=4680, heads=12, iters=5):
    n_slots = 13
    arena = torch.randn(n_slots, 2, T, heads*128, device="cuda").bfloat16()
    q = torch.randn(n_ent*T, heads*128, device="cuda").bfloat16()
    out = torch.empty_like(q)
    vis = [list(range(n_vis))]*n_ent
    b = N.make_batch(3, list(range(n_ent)), [0.0]*n_ent, [0]*n_ent, vis)
    mat = T*heads*128
    f = lambda: N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(arena), N.ptr(arena)+mat*2, 2*mat, T, b, T, heads, N.ptr(out), N.stream_ptr()), "a")
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)/iters
    fl = 4.0*n_ent*T*(n_vis*T)*heads*128
    print(f"entries={n_ent} vis_blocks={n_vis}: {ms:.3f} ms  {fl/ms/1e9:.0f} TFLOP/s")
for ne, nv in [(1,1),(1,8),(1,13),(5,13)]:
    run(ne, nv)
