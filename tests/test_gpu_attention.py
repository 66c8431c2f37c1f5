"""tcgen05 flash attention (csrc/attention.cu) vs a plain PyTorch fp32
softmax attention over the same bf16 inputs, with the reference gather order
(visible slots concatenated in the given order, denoiser.py:284-296).
Tolerance: rel-L2 <= 8e-3 (bf16 P and bf16 output; fp32 everywhere else)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2511_20426_b200 import _native as N


def run_attention(q, arena, vis, q_tokens, kv_tokens, heads):
    n = len(vis)
    out = torch.empty_like(q)
    b = N.make_batch(3, list(range(n)), [0.0] * n, [0] * n, vis)
    mat = kv_tokens * heads * 128
    N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(arena), N.ptr(arena) + mat * 2, 2 * mat,
                                       kv_tokens, b, q_tokens, heads, N.ptr(out), N.stream_ptr()),
            "attention")
    return out


def reference(q, arena, vis, q_tokens, heads):
    outs = []
    for e, slots in enumerate(vis):
        qe = q[e * q_tokens:(e + 1) * q_tokens].float().view(q_tokens, heads, 128)
        k = torch.cat([arena[s, 0] for s in slots]).float().view(-1, heads, 128)
        v = torch.cat([arena[s, 1] for s in slots]).float().view(-1, heads, 128)
        sc = torch.einsum("qhd,khd->hqk", qe, k) / 128 ** 0.5
        p = torch.softmax(sc, dim=-1)
        outs.append(torch.einsum("hqk,khd->qhd", p, v).reshape(q_tokens, heads * 128))
    return torch.cat(outs)


@pytest.mark.parametrize("q_tokens,kv_tokens,heads,vis", [
    (128, 128, 1, [[0]]),
    (200, 300, 2, [[0, 1, 2], [0, 1, 2, 3], [4]]),
    (384, 256, 2, [[5, 0, 3], [2]]),
    (192, 192, 2, [[0, 1, 2, 3, 4, 5]] * 5),
])
def test_attention_matches_torch(q_tokens, kv_tokens, heads, vis):
    g = torch.Generator(device="cuda").manual_seed(q_tokens + kv_tokens)
    n_slots = 6
    arena = (torch.randn(n_slots, 2, kv_tokens, heads * 128, device="cuda", generator=g)).bfloat16()
    q = (torch.randn(len(vis) * q_tokens, heads * 128, device="cuda", generator=g) * 2).bfloat16()
    got = run_attention(q, arena, vis, q_tokens, kv_tokens, heads)
    want = reference(q, arena, vis, q_tokens, heads)
    err = float((got.float() - want).norm() / want.norm())
    assert err < 8e-3, err


def test_attention_large_logits_rescale():
    """Growing row maxima across key tiles exercise the lazy O rescale."""
    g = torch.Generator(device="cuda").manual_seed(3)
    heads, T = 1, 512
    arena = torch.randn(4, 2, T, 128, device="cuda", generator=g)
    arena[:, 0] *= torch.linspace(0.1, 3.0, 4, device="cuda").view(4, 1, 1)   # later slots sharper
    arena = arena.bfloat16()
    q = (torch.randn(T, 128, device="cuda", generator=g) * 3).bfloat16()
    vis = [[0, 1, 2, 3]]
    got = run_attention(q, arena, vis, T, T, heads)
    want = reference(q, arena, vis, T, heads)
    assert float((got.float() - want).norm() / want.norm()) < 8e-3


def test_attention_deterministic_across_batching():
    """An entry's output does not depend on which other entries share the launch."""
    g = torch.Generator(device="cuda").manual_seed(5)
    heads, T = 2, 256
    arena = torch.randn(4, 2, T, heads * 128, device="cuda", generator=g).bfloat16()
    q = torch.randn(3 * T, heads * 128, device="cuda", generator=g).bfloat16()
    vis = [[0, 1], [0, 1, 2], [3, 0]]
    full = run_attention(q, arena, vis, T, T, heads)
    solo = run_attention(q[T:2 * T].contiguous(), arena, [vis[1]], T, T, heads)
    assert torch.equal(full[T:2 * T], solo)


@pytest.mark.parametrize("q_tokens,kv_tokens,heads,vis", [
    (4680, 256, 12, [[0, 1, 2], [0, 1, 2, 3], [4, 5, 0, 1, 2]]),   # ~5 items per CTA, mixed lengths
    (4680, 200, 12, [[0, 1, 2, 3, 4]] * 5),                       # bidirectional-like, ragged key tiles
    (1000, 384, 7, [[3], [0, 1]]),                                # fewer items than SMs
    (300, 128, 40, [[0, 1]] * 4),                                 # 14B head count
    (328, 256, 12, [[0, 1], [2, 3], [0, 1], [2, 3], [0, 1]]),    # last tiles paired across equal lists
])
def test_attention_balanced_kernel_bit_identical(q_tokens, kv_tokens, heads, vis):
    """The persistent balanced kernel (work lists of query-tile pairs and
    single tiles, barrier phases carried across items) gives bit-identical
    results to one CTA per (pair, entry, head), and matches torch."""
    g = torch.Generator(device="cuda").manual_seed(q_tokens + heads)
    arena = torch.randn(6, 2, kv_tokens, heads * 128, device="cuda", generator=g).bfloat16()
    q = (torch.randn(len(vis) * q_tokens, heads * 128, device="cuda", generator=g) * 2).bfloat16()
    try:
        N.lib().bc_attention_set_balance(0)
        grid = run_attention(q, arena, vis, q_tokens, kv_tokens, heads)
        N.lib().bc_attention_set_balance(1)
        bal = run_attention(q, arena, vis, q_tokens, kv_tokens, heads)
        again = run_attention(q, arena, vis, q_tokens, kv_tokens, heads)   # cached work list
    finally:
        N.lib().bc_attention_set_balance(1)
    assert torch.equal(grid, bal) and torch.equal(bal, again)
    if heads <= 12:
        want = reference(q, arena, vis, q_tokens, heads)
        assert float((bal.float() - want).norm() / want.norm()) < 8e-3
