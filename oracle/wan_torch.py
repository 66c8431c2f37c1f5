"""torch float32 restatement of oracle/wan.py -- TEST ORACLE ONLY.

The same Wan2.1-shaped DiT step as ``oracle/wan.py`` (numpy fp32, SURVEY.md
Appendix A), written one-to-one in torch so the checker can run at the
bench's full geometry (30 layers, 480x832, 512x4096 text) on the GPU in
seconds instead of hours on the host.  It is the checker, never the thing
measured: only ``tests/`` import it.

Numerics: every op is IEEE float32 with TF32 disabled (``exact_fp32``);
RoPE angles and the sinusoid are formed in float64 exactly as in
oracle/wan.py.  Weights are the device's bf16 values upcast on use (bf16 ->
fp32 is exact), so both sides see the same parameters.  Pinned to
oracle/wan.py at tiny geometry (tests/test_oracle_wan_torch.py, rel <= 1e-6)
and each sub-op to ``torch.nn.functional`` (layer_norm, rms_norm,
gelu(approximate="tanh"), scaled_dot_product_attention).

Conventions restated from the reference (file:line under
/root/reference/pkg/src/blockcascade): gather order = visible blocks
ascending, fresh batch KV wins (denoiser.py:284-296); RoPE time index =
global latent frame index (denoiser.py:247); sigma = level/1000, x0 = x_t -
sigma*v and renoise (1-s)*x0 + s*eps (denoiser.py:360-368).
"""

from __future__ import annotations

import contextlib
import math

import torch

EPS = 1e-6


@contextlib.contextmanager
def exact_fp32():
    """No TF32 anywhere inside (cuBLAS sgemm and cuDNN fp32 paths)."""
    m, c = torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32
    prec = torch.get_float32_matmul_precision()
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.set_float32_matmul_precision("highest")
    try:
        yield
    finally:
        torch.backends.cuda.matmul.allow_tf32 = m
        torch.backends.cudnn.allow_tf32 = c
        torch.set_float32_matmul_precision(prec)


# -- sub-operators (oracle/wan.py names) -------------------------------------

def layer_norm(x):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + EPS)


def rms_norm(x, w):
    return x / torch.sqrt((x * x).mean(-1, keepdim=True) + EPS) * w


def gelu_tanh(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def silu(x):
    return x / (1.0 + torch.exp(-x))


def sinusoid(t, freq_dim, device):
    half = freq_dim // 2
    w = torch.pow(torch.tensor(10000.0, dtype=torch.float64),
                  -torch.arange(half, dtype=torch.float64) / half)
    arg = t * w
    return torch.cat([torch.cos(arg), torch.sin(arg)]).float().to(device)


def rope_tables(frame0, frames, hp, wp, device):
    """float64 cos/sin per (token, pair); pairs [0,22) frame, [22,43) row,
    [43,64) column; D_part = 44/42/42 (oracle/wan.py rope_tables)."""
    kw = dict(dtype=torch.float64, device=device)
    f = torch.arange(frame0, frame0 + frames, **kw).repeat_interleave(hp * wp)
    h = torch.arange(hp, **kw).repeat_interleave(wp).repeat(frames)
    w = torch.arange(wp, **kw).repeat(frames * hp)
    inv_t = 1.0 / torch.pow(torch.tensor(10000.0, **kw), torch.arange(0, 44, 2, **kw) / 44)
    inv_h = 1.0 / torch.pow(torch.tensor(10000.0, **kw), torch.arange(0, 42, 2, **kw) / 42)
    ang = torch.cat([torch.outer(f, inv_t), torch.outer(h, inv_h), torch.outer(w, inv_h)], dim=1)
    return torch.cos(ang), torch.sin(ang)


def apply_rope(x, cos, sin):
    """x (T, H, 128) fp32; rotation in float64, result fp32."""
    T, H, _ = x.shape
    xr = x.reshape(T, H, 64, 2).double()
    c, s = cos[:, None, :], sin[:, None, :]
    out = torch.empty_like(xr)
    out[..., 0] = xr[..., 0] * c - xr[..., 1] * s
    out[..., 1] = xr[..., 0] * s + xr[..., 1] * c
    return out.reshape(T, H, 128).float()


def attention(q, k, v, heads, head_chunk=4, row_chunk=None):
    """q (Tq, d), k/v (Tk, d) fp32 -> (Tq, d): per head max-subtracted
    softmax(q k^T / sqrt(128)) v, all fp32 (sgemm)."""
    Tq, Tk = q.shape[0], k.shape[0]
    qh = q.reshape(Tq, heads, 128).transpose(0, 1)
    kh = k.reshape(Tk, heads, 128).transpose(0, 1)
    vh = v.reshape(Tk, heads, 128).transpose(0, 1)
    scale = 1.0 / math.sqrt(128.0)
    out = torch.empty((heads, Tq, 128), dtype=torch.float32, device=q.device)
    rc = row_chunk or Tq
    for h0 in range(0, heads, head_chunk):
        h1 = min(heads, h0 + head_chunk)
        kt = kh[h0:h1].transpose(1, 2)
        for r0 in range(0, Tq, rc):
            s = torch.matmul(qh[h0:h1, r0:r0 + rc], kt) * scale
            s -= s.amax(dim=-1, keepdim=True)
            p = torch.exp(s)
            p /= p.sum(dim=-1, keepdim=True)
            out[h0:h1, r0:r0 + rc] = torch.matmul(p, vh[h0:h1])
            del s, p
    return out.transpose(0, 1).reshape(Tq, heads * 128)


def patchify(x):
    F, C, H, W = x.shape
    t = x.reshape(F, C, H // 2, 2, W // 2, 2).permute(0, 2, 4, 1, 3, 5)
    return t.reshape(F * (H // 2) * (W // 2), C * 4)


def unpatchify(y, F, H, W):
    t = y.reshape(F, H // 2, W // 2, 2, 2, 16).permute(0, 5, 1, 3, 2, 4)
    return t.reshape(F, 16, H, W)


class WanTorchOracle:
    """``oracle.wan.WanOracle`` in torch fp32 on any device.  ``params``:
    name -> tensor (the product's bf16/fp32 device weights or numpy arrays);
    matrices are upcast to fp32 per use, never stored twice."""

    def __init__(self, params: dict, cfg, device=None):
        self.cfg = cfg
        self.d, self.L, self.H = cfg.model_dim, cfg.layers, cfg.heads
        first = next(iter(params.values()))
        self.device = torch.device(device) if device is not None else (
            first.device if isinstance(first, torch.Tensor) else torch.device("cpu"))
        self.p = {k: (v if isinstance(v, torch.Tensor) else torch.as_tensor(v)).to(self.device)
                  for k, v in params.items()}

    def w(self, name, layer=None):
        t = self.p[name] if layer is None else self.p[name][layer]
        return t.float()

    def linear(self, x, name, layer=None):
        return x @ self.w(name + "_w", layer).T + self.w(name + "_b", layer)

    def context(self, states):
        """Per-layer text (K, V) (fp32); ``states`` (text_len, text_dim)."""
        with exact_fp32():
            s = torch.as_tensor(states).to(self.device).float()
            h = gelu_tanh(s @ self.w("text_w1").T + self.w("text_b1"))
            ctx = h @ self.w("text_w2").T + self.w("text_b2")
            d, kv = self.d, []
            for l in range(self.L):
                t = ctx @ self.w("ckv_w", l).T + self.w("ckv_b", l)
                kv.append((rms_norm(t[:, :d], self.w("cnorm_k", l)), t[:, d:].contiguous()))
            return kv

    def time_embed(self, level):
        s = sinusoid(float(level), self.cfg.freq_dim, self.device)
        e = silu(s @ self.w("time_w1").T + self.w("time_b1")) @ self.w("time_w2").T + self.w("time_b2")
        e0 = silu(e) @ self.w("tproj_w").T + self.w("tproj_b")
        return e, e0.reshape(6, self.d)

    def forward(self, entries, pool_kv, visible, states=None, text_kv=None, keep_kv=True,
                taps=None):
        """entries: [(block, latents (S,D) or (S,16,H,W), level)];
        pool_kv: {block: [(K, V) per layer]} or {block: callable(layer) -> (K, V)};
        visible: {block: ascending visible blocks}.  Returns
        [(x0 (S,16,H,W) fp32, [(K, V) per layer] or None, v (S,16,H,W))].
        ``taps`` (optional dict) receives per-layer residual norms."""
        with exact_fp32(), torch.no_grad():
            return self._forward(entries, pool_kv, visible, states, text_kv, keep_kv, taps)

    def _forward(self, entries, pool_kv, visible, states, text_kv, keep_kv, taps):
        cfg, d, dev = self.cfg, self.d, self.device
        S, Hh, Ww = cfg.block_size, cfg.latent_height, cfg.latent_width
        hp, wp = Hh // 2, Ww // 2
        text_kv = text_kv if text_kv is not None else self.context(states)
        xs, X, temb, ropes = [], [], [], []
        for b, lat, level in entries:
            x = torch.as_tensor(lat).to(dev).float().reshape(S, 16, Hh, Ww)
            xs.append(x)
            X.append(patchify(x) @ self.w("patch_w").T + self.w("patch_b"))
            temb.append(self.time_embed(level))
            ropes.append(rope_tables(b * S, S, hp, wp, dev))
        kv_out = [[] for _ in entries]

        def pool_layer(vb, l):
            src = pool_kv[vb]
            k, v = src(l) if callable(src) else src[l]
            return (torch.as_tensor(k).to(dev).float().reshape(-1, d),
                    torch.as_tensor(v).to(dev).float().reshape(-1, d))

        for l in range(self.L):
            fresh, qs = {}, []
            mod_base = self.w("modulation", l)
            for i, (b, _, _) in enumerate(entries):
                mod = mod_base + temb[i][1]
                xn = layer_norm(X[i]) * (1 + mod[1]) + mod[0]
                qkv = xn @ self.w("qkv_w", l).T + self.w("qkv_b", l)
                q = rms_norm(qkv[:, :d], self.w("norm_q", l))
                k = rms_norm(qkv[:, d:2 * d], self.w("norm_k", l))
                v = qkv[:, 2 * d:].contiguous()
                c, s = ropes[i]
                q = apply_rope(q.reshape(-1, self.H, 128), c, s).reshape(-1, d)
                k = apply_rope(k.reshape(-1, self.H, 128), c, s).reshape(-1, d)
                fresh[b] = (k, v)
                qs.append(q)
                if keep_kv:
                    kv_out[i].append((k, v))
            for i, (b, _, _) in enumerate(entries):
                mod = mod_base + temb[i][1]
                ks, vs = [], []
                for vb in visible[b]:
                    kk, vv = fresh[vb] if vb in fresh else pool_layer(vb, l)
                    ks.append(kk)
                    vs.append(vv)
                att = attention(qs[i], torch.cat(ks), torch.cat(vs), self.H)
                del ks, vs
                X[i] = X[i] + mod[2] * (att @ self.w("o_w", l).T + self.w("o_b", l))
                xc = layer_norm(X[i]) * self.w("norm3_w", l) + self.w("norm3_b", l)
                qc = rms_norm(xc @ self.w("cq_w", l).T + self.w("cq_b", l), self.w("cnorm_q", l))
                ca = attention(qc, text_kv[l][0], text_kv[l][1], self.H)
                X[i] = X[i] + (ca @ self.w("co_w", l).T + self.w("co_b", l))
                xm = layer_norm(X[i]) * (1 + mod[4]) + mod[3]
                hmid = gelu_tanh(xm @ self.w("ffn1_w", l).T + self.w("ffn1_b", l))
                X[i] = X[i] + mod[5] * (hmid @ self.w("ffn2_w", l).T + self.w("ffn2_b", l))
                if taps is not None:
                    taps.setdefault(i, []).append(float(X[i].norm()))
            del fresh, qs
        outs = []
        hm = self.w("head_mod")
        for i, (b, _, level) in enumerate(entries):
            e = temb[i][0]
            xh = layer_norm(X[i]) * (1 + hm[1] + e) + hm[0] + e
            y = xh @ self.w("head_w").T + self.w("head_b")
            v = unpatchify(y, S, Hh, Ww)
            x0 = xs[i] - (level / 1000.0) * v
            outs.append((x0, kv_out[i] if keep_kv else None, v))
        return outs


def renoise(x0, eps, level):
    s = level / 1000.0
    return ((1.0 - s) * x0 + s * eps).float()
