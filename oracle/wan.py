"""numpy float32 restatement of the Wan2.1-shaped DiT step -- TEST ORACLE ONLY.

PARITY UNPINNED BY REFERENCE TESTS: the reference package has no Wan model
(SURVEY.md §8c).  This file restates the public Wan2.1 block (SURVEY.md
Appendix A) with the reference's conventions: RoPE time index = global
latent frame index (reference denoiser.py:247 position convention), key
gather order = visible blocks ascending (denoiser.py:284-296), noise
parameterisation sigma = level/1000 (denoiser.py:360-368).
Everything is float32 (weights are the device's bf16 values upcast); there
is no intermediate rounding, so it is the "fp32 reference" of the north
star's "bf16 vs fp32" tolerance.
"""

from __future__ import annotations

import numpy as np

EPS = 1e-6


def layer_norm(x):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    return (x - mu) / np.sqrt(var + EPS)


def rms_norm(x, w):
    return x / np.sqrt((x * x).mean(-1, keepdims=True) + EPS) * w


def gelu_tanh(x):
    return 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def silu(x):
    return x / (1.0 + np.exp(-x))


def sinusoid(t, freq_dim):
    half = freq_dim // 2
    w = np.power(10000.0, -np.arange(half, dtype=np.float64) / half)
    arg = t * w
    return np.concatenate([np.cos(arg), np.sin(arg)]).astype(np.float32)


def rope_tables(frame0, frames, hp, wp):
    """cos/sin per (token, pair) for head_dim 128: pairs [0,22) use the
    global frame index, [22,43) the patch row, [43,64) the patch column;
    inv_freq = 10000^(-2k/D_part) with D_part = 44/42/42 (Wan rope_params)."""
    f = np.repeat(np.arange(frame0, frame0 + frames), hp * wp)
    h = np.tile(np.repeat(np.arange(hp), wp), frames)
    w = np.tile(np.arange(wp), frames * hp)
    inv_t = 1.0 / np.power(10000.0, np.arange(0, 44, 2, dtype=np.float64) / 44)
    inv_h = 1.0 / np.power(10000.0, np.arange(0, 42, 2, dtype=np.float64) / 42)
    ang = np.concatenate([np.outer(f, inv_t), np.outer(h, inv_h), np.outer(w, inv_h)], axis=1)
    return np.cos(ang), np.sin(ang)


def apply_rope(x, cos, sin):
    """x: (T, H, 128); rotate complex pairs (2i, 2i+1)."""
    T, H, _ = x.shape
    xr = x.reshape(T, H, 64, 2).astype(np.float64)
    c, s = cos[:, None, :], sin[:, None, :]
    out = np.empty_like(xr)
    out[..., 0] = xr[..., 0] * c - xr[..., 1] * s
    out[..., 1] = xr[..., 0] * s + xr[..., 1] * c
    return out.reshape(T, H, 128).astype(np.float32)


def attention(q, k, v, heads, chunk=1024):
    """q (Tq, d), k/v (Tk, d) -> (Tq, d); softmax(q k^T / sqrt(128)) v per head."""
    Tq = q.shape[0]
    out = np.empty_like(q)
    qh = q.reshape(Tq, heads, 128)
    kh = k.reshape(-1, heads, 128)
    vh = v.reshape(-1, heads, 128)
    scale = np.float32(1.0 / np.sqrt(128.0))
    for h in range(heads):
        kt = kh[:, h, :].T.copy()
        vv = vh[:, h, :]
        for r0 in range(0, Tq, chunk):
            s = (qh[r0:r0 + chunk, h, :] @ kt) * scale
            s -= s.max(axis=1, keepdims=True)
            p = np.exp(s)
            p /= p.sum(axis=1, keepdims=True)
            out[r0:r0 + chunk, h * 128:(h + 1) * 128] = p @ vv
    return out


def patchify(x):
    """(F,16,H,W) -> (F*(H/2)*(W/2), 64), vector index c*4 + kh*2 + kw."""
    F, C, H, W = x.shape
    t = x.reshape(F, C, H // 2, 2, W // 2, 2).transpose(0, 2, 4, 1, 3, 5)
    return t.reshape(F * (H // 2) * (W // 2), C * 4)


def unpatchify(y, F, H, W):
    """(T, 64) with index (ph*2+pw)*16 + c -> (F,16,H,W)  (Wan unpatchify)."""
    t = y.reshape(F, H // 2, W // 2, 2, 2, 16).transpose(0, 5, 1, 3, 2, 4)
    return t.reshape(F, 16, H, W)


class WanOracle:
    def __init__(self, params: dict, cfg):
        self.p = {k: np.asarray(v, dtype=np.float32) for k, v in params.items()}
        self.cfg = cfg
        self.d = cfg.model_dim
        self.L = cfg.layers
        self.H = cfg.heads

    def linear(self, x, name, layer=None):
        w = self.p[name + "_w"] if layer is None else self.p[name + "_w"][layer]
        b = self.p[name + "_b"] if layer is None else self.p[name + "_b"][layer]
        return x @ w.T + b

    def context(self, states):
        p = self.p
        h = gelu_tanh(states.astype(np.float32) @ p["text_w1"].T + p["text_b1"])
        ctx = h @ p["text_w2"].T + p["text_b2"]
        d = self.d
        kv = []
        for l in range(self.L):
            t = ctx @ p["ckv_w"][l].T + p["ckv_b"][l]
            kv.append((rms_norm(t[:, :d], p["cnorm_k"][l]), t[:, d:]))
        return kv

    def time_embed(self, level):
        p = self.p
        s = sinusoid(float(level), self.cfg.freq_dim)
        e = silu(s @ p["time_w1"].T + p["time_b1"]) @ p["time_w2"].T + p["time_b2"]
        e0 = silu(e) @ p["tproj_w"].T + p["tproj_b"]
        return e.astype(np.float32), e0.reshape(6, self.d).astype(np.float32)

    def forward(self, entries, pool_kv, visible, states, text_kv=None):
        """entries: [(block, latents (S,D) or (S,16,H,W), level)];
        pool_kv: {block: [(K (T,d), V (T,d)) per layer]};
        visible: {block: ascending visible blocks}.
        Returns [(x0 (S,16,H,W) float32, [(K, V) per layer])]."""
        cfg, p, d = self.cfg, self.p, self.d
        S, Hh, Ww = cfg.block_size, cfg.latent_height, cfg.latent_width
        hp, wp = Hh // 2, Ww // 2
        text_kv = text_kv if text_kv is not None else self.context(states)
        xs, X, temb, ropes = [], [], [], []
        for b, lat, level in entries:
            x = np.asarray(lat, dtype=np.float32).reshape(S, 16, Hh, Ww)
            xs.append(x)
            X.append(patchify(x) @ p["patch_w"].T + p["patch_b"])
            temb.append(self.time_embed(level))
            ropes.append(rope_tables(b * S, S, hp, wp))
        kv_out = [[] for _ in entries]
        for l in range(self.L):
            fresh = {}
            qs = []
            for i, (b, _, _) in enumerate(entries):
                mod = p["modulation"][l] + temb[i][1]
                xn = layer_norm(X[i]) * (1 + mod[1]) + mod[0]
                qkv = xn @ p["qkv_w"][l].T + p["qkv_b"][l]
                q = rms_norm(qkv[:, :d], p["norm_q"][l])
                k = rms_norm(qkv[:, d:2 * d], p["norm_k"][l])
                v = qkv[:, 2 * d:]
                c, s = ropes[i]
                q = apply_rope(q.reshape(-1, self.H, 128), c, s).reshape(-1, d)
                k = apply_rope(k.reshape(-1, self.H, 128), c, s).reshape(-1, d)
                fresh[b] = (k, v)
                qs.append(q)
                kv_out[i].append((k, v))
            for i, (b, _, _) in enumerate(entries):
                mod = p["modulation"][l] + temb[i][1]
                ks, vs = [], []
                for vb in visible[b]:
                    kk, vv = fresh[vb] if vb in fresh else pool_kv[vb][l]
                    ks.append(kk)
                    vs.append(vv)
                att = attention(qs[i], np.concatenate(ks), np.concatenate(vs), self.H)
                X[i] = X[i] + mod[2] * (att @ p["o_w"][l].T + p["o_b"][l])
                xc = layer_norm(X[i]) * p["norm3_w"][l] + p["norm3_b"][l]
                qc = rms_norm(xc @ p["cq_w"][l].T + p["cq_b"][l], p["cnorm_q"][l])
                ca = attention(qc, text_kv[l][0], text_kv[l][1], self.H)
                X[i] = X[i] + (ca @ p["co_w"][l].T + p["co_b"][l])
                xm = layer_norm(X[i]) * (1 + mod[4]) + mod[3]
                hmid = gelu_tanh(xm @ p["ffn1_w"][l].T + p["ffn1_b"][l])
                X[i] = X[i] + mod[5] * (hmid @ p["ffn2_w"][l].T + p["ffn2_b"][l])
        outs = []
        for i, (b, _, level) in enumerate(entries):
            e = temb[i][0]
            xh = layer_norm(X[i]) * (1 + p["head_mod"][1] + e) + p["head_mod"][0] + e
            y = xh @ p["head_w"].T + p["head_b"]
            v = unpatchify(y, S, Hh, Ww)
            x0 = xs[i] - np.float32(level / 1000.0) * v
            outs.append((x0.astype(np.float32), kv_out[i]))
        return outs


def renoise(x0, eps, level):
    s = level / 1000.0
    return ((1.0 - s) * x0 + s * eps).astype(np.float32)
