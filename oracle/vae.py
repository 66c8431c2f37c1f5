"""torch float32 restatement of the Wan2.1 causal 3-D VAE decoder -- TEST ORACLE ONLY.

SURVEY.md §8(f) rank 1 ("VAE decode on a separate GPU").  The reference has
no VAE: its decode lane is a linear stand-in (reference
``pkg/src/blockcascade/executor.py:189-212``) timed by a cost model
(``engine.py:151-158``); the paper's streaming FPS includes decoding
(``PAPER.md:246``).  This file restates the *public* Wan2.1 VAE decoder
(Wan-Video/Wan2.1 ``wan/modules/vae.py``: ``CausalConv3d``, ``RMS_norm``,
``Resample``, ``ResidualBlock``, ``AttentionBlock``, ``Decoder3d``,
``WanVAE_.decode``) from its published definition -- no third-party copy
of it is installed here, so this restatement is PARITY UNPINNED against
an external implementation; each sub-op is checked against
``torch.nn.functional`` (conv3d/conv2d/normalize/interpolate/SDPA) by
construction and in tests/test_oracle_vae.py.

It is the checker, never the thing measured: only ``tests/`` (and the
bench's CPU leg) import it.  It decodes exactly the way Wan streams: ONE
latent frame per decoder call with the per-conv feature caches
(``CACHE_T = 2``) and the ``'Rep'`` first-chunk rule of ``upsample3d``,
so the product's block-at-a-time decode (3 latent frames per call) is
checked against the frame-at-a-time reference semantics.

Parameters are a flat dict ``name -> float32 tensor`` in torch conv layouts
(``[Cout, Cin, kt, kh, kw]``); names follow ``layer_specs``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

CACHE_T = 2

# Wan2.1 VAE latent statistics (wan/modules/vae.py, WanVAE.__init__): the
# decoder input is z * std + mean per channel.
LATENT_MEAN = (-0.7571, -0.7089, -0.9113, 0.1075, -0.1745, 0.9653, -0.1517, 1.5508,
               0.4134, -0.0715, 0.5517, -0.3632, -0.1922, -0.9497, 0.2503, -0.2921)
LATENT_STD = (2.8184, 1.4541, 2.3275, 2.6558, 1.2196, 1.7708, 2.6052, 2.0743,
              3.2687, 2.1526, 2.8652, 1.5579, 1.6382, 1.1253, 2.8251, 1.9160)


@dataclass(frozen=True)
class VaeDims:
    dim: int = 96
    z_dim: int = 16
    dim_mult: tuple = (1, 2, 4, 4)
    num_res_blocks: int = 2
    temperal_upsample: tuple = (True, True, False)   # = temperal_downsample[::-1]


def layer_specs(d: VaeDims):
    """Decoder3d.__init__ restated: the ordered layer list.
    ('res', name, cin, cout) | ('attn', name, c) | ('up3d'|'up2d', name, c)."""
    dims = [d.dim * u for u in (d.dim_mult[-1],) + tuple(d.dim_mult[::-1])]
    out = [("res", "mid0", dims[0], dims[0]), ("attn", "mid1", dims[0]), ("res", "mid2", dims[0], dims[0])]
    k = 0
    out_dim = dims[0]
    for i, (in_dim, out_dim) in enumerate(zip(dims[:-1], dims[1:])):
        if i in (1, 2, 3):
            in_dim = in_dim // 2
        for _ in range(d.num_res_blocks + 1):
            out.append(("res", f"up{k}", in_dim, out_dim))
            k += 1
            in_dim = out_dim
        if i != len(d.dim_mult) - 1:
            out.append(("up3d" if d.temperal_upsample[i] else "up2d", f"up{k}", out_dim))
            k += 1
    return dims, out, out_dim


def param_shapes(d: VaeDims) -> dict:
    """name -> (torch shape, fan_in or None, kind) ; kind in w / b / g."""
    dims, specs, last = layer_specs(d)
    z = d.z_dim
    p = {"conv2.w": ((z, z, 1, 1, 1), z, "w"), "conv2.b": ((z,), None, "b"),
         "conv1.w": ((dims[0], z, 3, 3, 3), z * 27, "w"), "conv1.b": ((dims[0],), None, "b")}
    for s in specs:
        if s[0] == "res":
            _, n, ci, co = s
            p[f"{n}.n1"] = ((ci,), None, "g")
            p[f"{n}.c1.w"] = ((co, ci, 3, 3, 3), ci * 27, "w")
            p[f"{n}.c1.b"] = ((co,), None, "b")
            p[f"{n}.n2"] = ((co,), None, "g")
            p[f"{n}.c2.w"] = ((co, co, 3, 3, 3), co * 27, "w")
            p[f"{n}.c2.b"] = ((co,), None, "b")
            if ci != co:
                p[f"{n}.sc.w"] = ((co, ci, 1, 1, 1), ci, "w")
                p[f"{n}.sc.b"] = ((co,), None, "b")
        elif s[0] == "attn":
            _, n, c = s
            p[f"{n}.norm"] = ((c,), None, "g")
            p[f"{n}.qkv.w"] = ((3 * c, c, 1, 1), c, "w")
            p[f"{n}.qkv.b"] = ((3 * c,), None, "b")
            p[f"{n}.proj.w"] = ((c, c, 1, 1), c, "w")   # Wan zero-inits this; random here
            p[f"{n}.proj.b"] = ((c,), None, "b")
        else:
            _, n, c = s
            p[f"{n}.rs.w"] = ((c // 2, c, 3, 3), c * 9, "w")
            p[f"{n}.rs.b"] = ((c // 2,), None, "b")
            if s[0] == "up3d":
                p[f"{n}.tc.w"] = ((2 * c, c, 3, 1, 1), c * 3, "w")
                p[f"{n}.tc.b"] = ((2 * c,), None, "b")
    p["head.n"] = ((last,), None, "g")
    p["head.w"] = ((3, last, 3, 3, 3), last * 27, "w")
    p["head.b"] = ((3,), None, "b")
    return p


# -- sub-operators (Wan names) ----------------------------------------------

def causal_conv3d(x, w, b, cache=None):
    """CausalConv3d.forward: causal time padding 2*pad_t in front (less the
    cached frames), symmetric spatial padding.  x [B, C, T, H, W]."""
    kt, kh, kw = w.shape[2:]
    pt, ph, pw = (kt - 1) // 2, (kh - 1) // 2, (kw - 1) // 2
    padding = [pw, pw, ph, ph, 2 * pt, 0]
    if cache is not None and 2 * pt > 0:
        x = torch.cat([cache, x], dim=2)
        padding[4] -= cache.shape[2]
    x = F.pad(x, padding)
    return F.conv3d(x, w, b)


def rms_norm(x, g):
    """RMS_norm (channel_first): F.normalize over C * sqrt(C) * gamma."""
    c = x.shape[1]
    shape = (1, c) + (1,) * (x.dim() - 2)
    return F.normalize(x, dim=1) * math.sqrt(c) * g.view(shape)


def _cache_after(x, old):
    """The cache update every cached conv does: the last CACHE_T input frames,
    topped up with the previous cache's last frame for 1-frame chunks."""
    c = x[:, :, -CACHE_T:].clone()
    if c.shape[2] < 2 and old is not None:
        c = torch.cat([old[:, :, -1:], c], dim=2)
    return c


class _Cache:
    def __init__(self):
        self.feat = {}


def _cconv(x, w, b, key, cache: _Cache):
    old = cache.feat.get(key)
    new = _cache_after(x, old)
    y = causal_conv3d(x, w, b, old)
    cache.feat[key] = new
    return y


def residual_block(x, P, n, cache):
    h = causal_conv3d(x, P[f"{n}.sc.w"], P[f"{n}.sc.b"]) if f"{n}.sc.w" in P else x
    y = F.silu(rms_norm(x, P[f"{n}.n1"]))
    y = _cconv(y, P[f"{n}.c1.w"], P[f"{n}.c1.b"], f"{n}.c1", cache)
    y = F.silu(rms_norm(y, P[f"{n}.n2"]))
    y = _cconv(y, P[f"{n}.c2.w"], P[f"{n}.c2.b"], f"{n}.c2", cache)
    return y + h


def attention_block(x, P, n):
    """AttentionBlock: per-frame single-head attention over H*W tokens."""
    identity = x
    b, c, t, h, w = x.shape
    y = x.permute(0, 2, 1, 3, 4).reshape(b * t, c, h, w)
    y = rms_norm(y, P[f"{n}.norm"])
    qkv = F.conv2d(y, P[f"{n}.qkv.w"], P[f"{n}.qkv.b"])
    q, k, v = qkv.reshape(b * t, 1, 3 * c, h * w).permute(0, 1, 3, 2).contiguous().chunk(3, dim=-1)
    y = F.scaled_dot_product_attention(q, k, v)
    y = y.squeeze(1).permute(0, 2, 1).reshape(b * t, c, h, w)
    y = F.conv2d(y, P[f"{n}.proj.w"], P[f"{n}.proj.b"])
    return y.reshape(b, t, c, h, w).permute(0, 2, 1, 3, 4) + identity


def resample(x, P, n, mode, cache):
    """Resample(mode='upsample2d'|'upsample3d') with Wan's first-chunk 'Rep'
    rule: the first chunk of the stream is not time-upsampled, and the time
    conv of the second chunk pads with zeros instead of a cache."""
    b, c, t, h, w = x.shape
    if mode == "up3d":
        key = f"{n}.tc"
        old = cache.feat.get(key)
        if old is None:
            cache.feat[key] = "Rep"
        else:
            new = x[:, :, -CACHE_T:].clone()
            if new.shape[2] < 2 and isinstance(old, str):
                new = torch.cat([torch.zeros_like(new), new], dim=2)
            elif new.shape[2] < 2:
                new = torch.cat([old[:, :, -1:], new], dim=2)
            if isinstance(old, str):
                x = causal_conv3d(x, P[f"{key}.w"], P[f"{key}.b"])
            else:
                x = causal_conv3d(x, P[f"{key}.w"], P[f"{key}.b"], old)
            cache.feat[key] = new
            x = x.reshape(b, 2, c, t, h, w)
            x = torch.stack((x[:, 0], x[:, 1]), 3)
            x = x.reshape(b, c, t * 2, h, w)
    t = x.shape[2]
    y = x.permute(0, 2, 1, 3, 4).reshape(b * t, c, h, w)
    y = F.interpolate(y, scale_factor=(2.0, 2.0), mode="nearest-exact")
    y = F.conv2d(y, P[f"{n}.rs.w"], P[f"{n}.rs.b"], padding=1)
    return y.reshape(b, t, c // 2, 2 * h, 2 * w).permute(0, 2, 1, 3, 4)


def decoder_chunk(x, P, d: VaeDims, cache: _Cache):
    """Decoder3d.forward over one chunk x [1, z, t, h, w] (after conv2)."""
    _, specs, _ = layer_specs(d)
    x = _cconv(x, P["conv1.w"], P["conv1.b"], "conv1", cache)
    for s in specs:
        if s[0] == "res":
            x = residual_block(x, P, s[1], cache)
        elif s[0] == "attn":
            x = attention_block(x, P, s[1])
        else:
            x = resample(x, P, s[1], s[0], cache)
    y = F.silu(rms_norm(x, P["head.n"]))
    return _cconv(y, P["head.w"], P["head.b"], "head", cache)


class VaeDecoderOracle:
    """Streaming decoder with Wan's per-conv feature caches.  ``decode(z)``
    takes latents [16, T, h, w] (float32, normalised like Wan's) and returns
    the video [3, n, 8h, 8w] clamped to [-1, 1]; successive calls continue
    the stream (block after block), one latent frame per decoder call."""

    def __init__(self, params: dict, dims: VaeDims = VaeDims()):
        self.P = params
        self.d = dims
        self.cache = _Cache()
        dev = params["conv1.w"].device
        self.mean = torch.tensor(LATENT_MEAN, dtype=torch.float32, device=dev).view(1, -1, 1, 1, 1)
        self.std = torch.tensor(LATENT_STD, dtype=torch.float32, device=dev).view(1, -1, 1, 1, 1)

    def reset(self):
        self.cache = _Cache()

    def decode(self, z, frame_by_frame: bool = True):
        z = z.unsqueeze(0).float()
        z = z / (1.0 / self.std) + self.mean          # WanVAE_.decode: z / scale[1] + scale[0]
        x = causal_conv3d(z, self.P["conv2.w"], self.P["conv2.b"])
        if frame_by_frame:
            outs = [decoder_chunk(x[:, :, i:i + 1], self.P, self.d, self.cache) for i in range(x.shape[2])]
            out = torch.cat(outs, 2)
        else:
            out = decoder_chunk(x, self.P, self.d, self.cache)
        return out.clamp(-1.0, 1.0)[0]


def random_params(dims: VaeDims, seed: int = 11, device="cpu") -> dict:
    """Deterministic random init in the oracle's own layouts (tests that do
    not go through the product's weights)."""
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    out = {}
    for name, (shape, fan_in, kind) in param_shapes(dims).items():
        r = torch.randn(shape, generator=g)
        if kind == "w":
            t = r / math.sqrt(fan_in)
        elif kind == "b":
            t = 0.02 * r
        else:
            t = 1.0 + 0.05 * r
        out[name] = t.to(device)
    return out
