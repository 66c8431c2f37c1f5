"""numpy float64 restatement of the reference toy DiT -- TEST ORACLE ONLY.

Each function cites the reference function it restates
(/root/reference/pkg/src/blockcascade/denoiser.py).  Pinned bit-for-bit
against the reference's own outputs (tests/golden/toy_golden.npz).
"""

from __future__ import annotations

import numpy as np

LEVEL_FEATS = 8      # denoiser.py:25
RMS_EPS = 1e-6       # denoiser.py:26


def weights_from(w):
    """Accept either package's ModelWeights (same field names)."""
    return dict(w_in=w.w_in, w_cond=w.w_cond, w_level=w.w_level, w_q=w.w_q, w_k=w.w_k,
                w_v=w.w_v, w_o=w.w_o, w_head=w.w_head, heads=w.heads)


def position_encoding(frame0, size, dim):
    """denoiser.py:214-221 -- interleaved sin/cos of pos / 10000^(2i/dim)."""
    pos = np.arange(frame0, frame0 + size, dtype=np.float64)[:, None]
    i = np.arange(dim // 2, dtype=np.float64)[None, :]
    ang = pos / np.power(10000.0, 2.0 * i / dim)
    enc = np.zeros((size, dim))
    enc[:, 0::2] = np.sin(ang)
    enc[:, 1::2] = np.cos(ang)
    return enc


def level_features(level):
    """denoiser.py:224-227."""
    s = level / 1000.0
    k = np.arange(1, LEVEL_FEATS // 2 + 1, dtype=np.float64)
    return np.concatenate([np.sin(2 * np.pi * s * k), np.cos(2 * np.pi * s * k)])


def rms_norm(h):
    """denoiser.py:230-231."""
    return h / np.sqrt(np.mean(h * h, axis=-1, keepdims=True) + RMS_EPS)


def embed(W, block, latents, level, cond_emb):
    """denoiser.py:234-250 (validation omitted; the product validates)."""
    s, d = latents.shape
    h = latents @ W["w_in"].T
    h += position_encoding(block * s, s, d)
    h += W["w_level"] @ level_features(level)
    h += W["w_cond"] @ cond_emb
    return h


def qkv(W, layer, h):
    """denoiser.py:253-261."""
    s, d = h.shape
    hd = d // W["heads"]
    hn = rms_norm(h)
    shape = (s, W["heads"], hd)
    return ((hn @ W["w_q"][layer].T).reshape(shape), (hn @ W["w_k"][layer].T).reshape(shape),
            (hn @ W["w_v"][layer].T).reshape(shape))


def attend(W, layer, h, q, keys, values):
    """denoiser.py:264-277 -- per-head max-subtracted softmax, then O-proj."""
    s, d = h.shape
    H = W["heads"]
    hd = d // H
    out = np.empty((s, H, hd))
    for head in range(H):
        sc = (q[:, head, :] @ keys[:, head, :].T) * (1.0 / np.sqrt(hd))
        sc -= sc.max(axis=1, keepdims=True)
        p = np.exp(sc)
        p /= p.sum(axis=1, keepdims=True)
        out[:, head, :] = p @ values[:, head, :]
    return h + out.reshape(s, d) @ W["w_o"][layer].T


def head(W, h):
    """denoiser.py:280-281."""
    return rms_norm(h) @ W["w_head"].T


def forward(W, entries, pool_kv, visible):
    """denoiser.py:299-357 without validation.

    entries: list of (block, latents (S,D), level, cond_emb)
    pool_kv: {block: [(keys, values) per layer]}
    visible: {block: ascending visible key blocks}  (build_mask semantics)
    Returns [(x0, [(keys, values) per layer])] in entry order.
    """
    L = W["w_q"].shape[0]
    hidden = [embed(W, b, x, lvl, c) for b, x, lvl, c in entries]
    kv_out = [[] for _ in entries]
    for layer in range(L):
        fresh = [qkv(W, layer, h) for h in hidden]
        by_block = {e[0]: (f[1], f[2]) for e, f in zip(entries, fresh)}
        new_hidden = []
        for i, (b, _, _, _) in enumerate(entries):
            ks, vs = [], []
            for vb in visible[b]:                  # _gather, denoiser.py:284-296
                k, v = by_block[vb] if vb in by_block else pool_kv[vb][layer]
                ks.append(k)
                vs.append(v)
            new_hidden.append(attend(W, layer, hidden[i], fresh[i][0],
                                     np.concatenate(ks), np.concatenate(vs)))
        hidden = new_hidden
        for i, f in enumerate(fresh):
            kv_out[i].append((f[1], f[2]))
    return [(head(W, h), kv) for h, kv in zip(hidden, kv_out)]


def renoise(x0, eps, level):
    """denoiser.py:360-368."""
    s = level / 1000.0
    return (1.0 - s) * x0 + s * eps
