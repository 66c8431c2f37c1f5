"""Wan2.1-shaped causal VAE decode on the device.

The reference's decode lane is a cost-model charge (``engine.py:151-158``,
``decode_overlap`` on a second worker) over a linear stand-in
(``executor.py:189-212``, kept here as ``executor.decode_block``).  The
paper's streaming FPS includes decoding and puts it on a side GPU
(``PAPER.md:37``, ``PAPER.md:246``).  This module decodes the blocks the
cascade emits with the public Wan2.1 VAE decoder architecture
(``Decoder3d``: conv1 -> middle {ResidualBlock, AttentionBlock,
ResidualBlock} -> 4 upsample stages of 3 ResidualBlocks with two temporal
and three spatial x2 resamples -> RMS_norm/SiLU/CausalConv3d head), random
init, streamed block after block with Wan's causal feature caches.

Every op runs in ``libbcb200.so`` (``csrc/vae.cu``: the tcgen05
implicit-GEMM causal conv with fused norm/SiLU/residual epilogues, the
resample / attention helpers; ``gemm.cu`` for the per-frame attention
GEMMs).  Torch owns the buffers and does the history copies (plumbing).

Layout: every activation is "padded frames" ``[n_frames][H+2][W+2][C]``
channels-last with a zero border; frames 0-1 of a causal conv input hold
that conv's cache (its last two input frames of the previous block, zero
before the first).  A block's frames live at frames 2 .. 2+T-1.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from . import _native as N
from .errors import ContractViolation

LATENT_MEAN = (-0.7571, -0.7089, -0.9113, 0.1075, -0.1745, 0.9653, -0.1517, 1.5508,
               0.4134, -0.0715, 0.5517, -0.3632, -0.1922, -0.9497, 0.2503, -0.2921)
LATENT_STD = (2.8184, 1.4541, 2.3275, 2.6558, 1.2196, 1.7708, 2.6052, 2.0743,
              3.2687, 2.1526, 2.8652, 1.5579, 1.6382, 1.1253, 2.8251, 1.9160)


@dataclass(frozen=True)
class VaeConfig:
    dim: int = 96                      # Wan2.1 VAE base width
    z_dim: int = 16
    dim_mult: tuple = (1, 2, 4, 4)
    num_res_blocks: int = 2
    temporal_upsample: tuple = (True, True, False)
    latent_h: int = 60                 # 480 x 832 video
    latent_w: int = 104
    block_size: int = 3                # latent frames per decode call

    @property
    def video_h(self) -> int:
        return self.latent_h * 8

    @property
    def video_w(self) -> int:
        return self.latent_w * 8

    def frames_out(self, n_latent: int, first: bool) -> int:
        """Video frames a block of n latent frames decodes to (Wan: the
        stream's first latent frame gives 1 frame, every other gives 4)."""
        return 1 + 4 * (n_latent - 1) if first else 4 * n_latent


def vae_config(name: str = "wan2.1", **kw) -> VaeConfig:
    if name == "wan2.1":
        return VaeConfig(**kw)
    if name == "tiny":
        base = dict(dim=32, latent_h=8, latent_w=12)
        base.update(kw)
        return VaeConfig(**base)
    raise ContractViolation(f"unknown VAE preset {name!r}")


def layer_specs(cfg: VaeConfig):
    """Decoder3d's layer list (Wan2.1 ``vae.py``): ('res', name, cin, cout),
    ('attn', name, c), ('up3d' | 'up2d', name, c)."""
    dims = [cfg.dim * u for u in (cfg.dim_mult[-1],) + tuple(cfg.dim_mult[::-1])]
    out = [("res", "mid0", dims[0], dims[0]), ("attn", "mid1", dims[0]), ("res", "mid2", dims[0], dims[0])]
    k = 0
    out_dim = dims[0]
    for i, (in_dim, out_dim) in enumerate(zip(dims[:-1], dims[1:])):
        if i in (1, 2, 3):
            in_dim //= 2
        for _ in range(cfg.num_res_blocks + 1):
            out.append(("res", f"up{k}", in_dim, out_dim))
            k += 1
            in_dim = out_dim
        if i != len(cfg.dim_mult) - 1:
            out.append(("up3d" if cfg.temporal_upsample[i] else "up2d", f"up{k}", out_dim))
            k += 1
    return dims, out, out_dim


def param_shapes(cfg: VaeConfig) -> dict:
    """name -> (torch conv shape, fan_in, kind) -- the same names and layouts
    as the checker (oracle/vae.py)."""
    dims, specs, last = layer_specs(cfg)
    z = cfg.z_dim
    p = {"conv2.w": ((z, z, 1, 1, 1), z, "w"), "conv2.b": ((z,), None, "b"),
         "conv1.w": ((dims[0], z, 3, 3, 3), z * 27, "w"), "conv1.b": ((dims[0],), None, "b")}
    for s in specs:
        if s[0] == "res":
            _, n, ci, co = s
            p.update({f"{n}.n1": ((ci,), None, "g"), f"{n}.c1.w": ((co, ci, 3, 3, 3), ci * 27, "w"),
                      f"{n}.c1.b": ((co,), None, "b"), f"{n}.n2": ((co,), None, "g"),
                      f"{n}.c2.w": ((co, co, 3, 3, 3), co * 27, "w"), f"{n}.c2.b": ((co,), None, "b")})
            if ci != co:
                p[f"{n}.sc.w"] = ((co, ci, 1, 1, 1), ci, "w")
                p[f"{n}.sc.b"] = ((co,), None, "b")
        elif s[0] == "attn":
            _, n, c = s
            p.update({f"{n}.norm": ((c,), None, "g"), f"{n}.qkv.w": ((3 * c, c, 1, 1), c, "w"),
                      f"{n}.qkv.b": ((3 * c,), None, "b"), f"{n}.proj.w": ((c, c, 1, 1), c, "w"),
                      f"{n}.proj.b": ((c,), None, "b")})
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


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


class VaeWeights:
    """Random-init decoder weights.  ``params``: fp32 torch-layout tensors
    (conv weights hold bf16-representable values -- what the device uses);
    ``dev``: the kernels' layouts (conv weights bf16 [cout][taps][cin],
    cin padded to 32, cout padded to 16)."""

    def __init__(self, cfg: VaeConfig, params: dict, seed: int):
        torch = N.torch_mod()
        self.cfg, self.params, self.seed = cfg, params, seed
        dev = {}
        for name, t in params.items():
            if name.endswith(".w") and t.dim() >= 4 and name != "conv2.w":
                w = t if t.dim() == 5 else t.unsqueeze(2)            # 2-D conv -> kt = 1
                co, ci = w.shape[0], w.shape[1]
                co_p, ci_p = _round_up(co, 16), _round_up(ci, 32)
                k = w.permute(0, 2, 3, 4, 1).reshape(co, -1, ci)       # [cout][taps][cin]
                full = torch.zeros((co_p, k.shape[1], ci_p), dtype=torch.bfloat16, device="cuda")
                full[:co, :, :ci] = k.bfloat16()
                dev[name] = full.reshape(co_p, -1).contiguous()
            elif name.endswith(".b") and name.replace(".b", ".w") in params and name != "conv2.b":
                co_p = _round_up(t.numel(), 16)
                b = torch.zeros(co_p, dtype=torch.float32, device="cuda")
                b[:t.numel()] = t
                dev[name] = b
            else:
                dev[name] = t.float().contiguous()
        dev["conv2.w"] = params["conv2.w"].reshape(cfg.z_dim, cfg.z_dim).float().contiguous()
        dev["latent_mean"] = torch.tensor(LATENT_MEAN, dtype=torch.float32, device="cuda")
        dev["latent_std"] = torch.tensor(LATENT_STD, dtype=torch.float32, device="cuda")
        self.dev = dev

    @classmethod
    def random(cls, cfg: VaeConfig, seed: int = 11) -> "VaeWeights":
        torch = N.torch_mod()
        gen = torch.Generator(device="cuda")
        gen.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
        params = {}
        for name, (shape, fan_in, kind) in param_shapes(cfg).items():
            r = torch.randn(shape, generator=gen, device="cuda")
            if kind == "w":
                t = (r / math.sqrt(fan_in)).bfloat16().float()
            elif kind == "b":
                t = 0.02 * r
            else:
                t = 1.0 + 0.05 * r
            params[name] = t.contiguous()
        return cls(cfg, params, seed)

    def host_params(self, device="cpu") -> dict:
        """fp32 torch-layout copies for the checker."""
        return {k: v.detach().to(device).float().clone() for k, v in self.params.items()}


class _Level:
    def __init__(self, h, w, frames):
        self.h, self.w, self.frames = h, w, frames
        self.F = (h + 2) * (w + 2)

    def buf(self, torch, c, dtype):
        return torch.zeros((self.frames, self.h + 2, self.w + 2, c), dtype=dtype, device="cuda")


class VaeDecoder:
    """Streaming decoder: ``decode_block(z)`` takes one emitted block's
    latents [T][16][h][w] (fp32, device) and returns its video frames
    [n][3][8h][8w] (fp32, device, clamped to [-1, 1]); consecutive calls
    continue the stream with Wan's causal caches.  All work is enqueued on
    ``stream`` (default: a private side stream, so decoding overlaps the
    next cascade iteration)."""

    def __init__(self, weights: VaeWeights, stream=None):
        torch = N.torch_mod()
        self.torch = torch
        self.w = weights
        cfg = self.cfg = weights.cfg
        if cfg.block_size < 2:
            raise ContractViolation("VAE decode needs >= 2 latent frames per block (causal cache of 2)")
        self.stream = stream if stream is not None else torch.cuda.Stream()
        self.dims, self.specs, self.last = layer_specs(cfg)
        T = cfg.block_size
        t_out = [T]
        for s in self.specs:
            if s[0] == "up3d":
                t_out.append(2 * t_out[-1])
            elif s[0] == "up2d":
                t_out.append(t_out[-1])
        self.levels = [_Level(cfg.latent_h << i, cfg.latent_w << i, 2 + t) for i, t in enumerate(t_out)]
        self.T_max = t_out
        self._alloc()
        self.first = True
        self.launches = 0
        self._prof = None                 # list of (label, flops, end event) when profiling

    def profile(self, on: bool = True):
        """Per-op CUDA events on the decode stream (adds a sync-free event per
        op); ``profile_report()`` folds them into per-label ms / TFLOP/s."""
        self._prof = [] if on else None
        if on:
            ev = self.torch.cuda.Event(enable_timing=True)
            ev.record(self.stream)
            self._prof.append(("start", 0.0, ev))

    def _mark(self, label, flops=0.0):
        if self._prof is not None:
            ev = self.torch.cuda.Event(enable_timing=True)
            ev.record(self.stream)
            self._prof.append((label, flops, ev))

    def profile_report(self) -> dict:
        self.torch.cuda.synchronize()
        out = {}
        prof = self._prof or []
        for (_, _, e0), (label, fl, e1) in zip(prof[:-1], prof[1:]):
            ms = e0.elapsed_time(e1)
            d = out.setdefault(label, [0.0, 0.0, 0])
            d[0] += ms
            d[1] += fl
            d[2] += 1
        self.profile(self._prof is not None)
        return {k: {"ms": v[0], "tflops": (v[1] / v[0] / 1e9 if v[0] > 0 else 0.0), "n": v[2]} for k, v in out.items()}

    # -- buffers ----------------------------------------------------------
    def _alloc(self):
        torch = self.torch
        bf, f32 = torch.bfloat16, torch.float32
        L = self.levels
        self._scr = {}
        self.hist = []                    # (buffer, level) of every causal (kt = 3) conv input
        self.prep = L[0].buf(torch, 32, bf)
        self.hist.append((self.prep, 0))
        self.x = {}                       # level -> {channels: fp32 residual stream}
        self.raw = {}                     # level -> {channels: bf16 raw x (shortcut / time-conv input)}
        self.in1, self.in2 = {}, {}
        self.tc_out, self.up_in = {}, {}
        lvl = 0
        for s in self.specs:
            if s[0] == "res":
                _, n, ci, co = s
                for c in (ci, co):
                    self.x.setdefault(lvl, {}).setdefault(c, L[lvl].buf(torch, c, f32))
                self.in1[n] = L[lvl].buf(torch, ci, bf)
                self.in2[n] = L[lvl].buf(torch, co, bf)
                self.hist += [(self.in1[n], lvl), (self.in2[n], lvl)]
                if ci != co:
                    self.raw.setdefault(lvl, {}).setdefault(ci, L[lvl].buf(torch, ci, bf))
            elif s[0] == "attn":
                _, n, c = s
                h, w = L[lvl].h, L[lvl].w
                self.np_tok = _round_up(h * w, 128)
                self.attn_in = L[lvl].buf(torch, c, bf)
                self.qkv = L[lvl].buf(torch, 3 * c, bf)
                self.aq = torch.zeros((self.np_tok, c), dtype=bf, device="cuda")
                self.ak = torch.zeros((self.np_tok, c), dtype=bf, device="cuda")
                self.avt = torch.zeros((c, self.np_tok), dtype=bf, device="cuda")
                self.aS = torch.empty((h * w, self.np_tok), dtype=f32, device="cuda")
                self.aP = torch.empty((h * w, self.np_tok), dtype=bf, device="cuda")
                self.aO = torch.empty((h * w, c), dtype=bf, device="cuda")
                self.aproj = torch.empty((h * w, c), dtype=f32, device="cuda")
            else:
                _, n, c = s
                if s[0] == "up3d":
                    self.raw.setdefault(lvl, {}).setdefault(c, L[lvl].buf(torch, c, bf))
                    self.hist.append((self.raw[lvl][c], lvl))
                    self.tc_out[n] = L[lvl].buf(torch, 2 * c, f32)
                lvl += 1
                self.up_in[n] = L[lvl].buf(torch, c, bf)
                self.x.setdefault(lvl, {}).setdefault(c // 2, L[lvl].buf(torch, c // 2, f32))
        self.head_in = L[lvl].buf(torch, self.last, bf)
        self.hist.append((self.head_in, lvl))

    def nbytes(self) -> int:
        seen, total = set(), 0
        for t in [self.prep, self.head_in, self.attn_in, self.qkv, self.aq, self.ak, self.avt, self.aS, self.aP,
                  self.aO, self.aproj] + list(self.in1.values()) + list(self.in2.values()) + \
                 list(self.tc_out.values()) + list(self.up_in.values()) + \
                 [b for d in self.x.values() for b in d.values()] + [b for d in self.raw.values() for b in d.values()]:
            if id(t) not in seen:
                seen.add(id(t))
                total += t.numel() * t.element_size()
        return total

    def reset(self):
        """Start a new video: zero every cache (and border)."""
        with self.torch.cuda.stream(self.stream):
            for b, _ in self.hist:
                b.zero_()
        self.first = True

    # -- ops --------------------------------------------------------------
    def _conv(self, lvl, T, inp, wname, bname, kt, kh, kw, frame0=2, res=None, out32=None, out16=None,
              act=None, gamma=None, silu=1, video=None, video_ch=0):
        L = self.levels[lvl]
        w = self.w.dev[wname]
        split_norm = act is not None and w.shape[0] > 192 and w.shape[0] % 192 == 0
        if split_norm:                      # row wider than one unit: norm in a second pass
            if out32 is None:
                out32 = self._scratch(lvl, w.shape[0])
            act_buf, act = act, None
        a = N.VaeConvArgs()
        a.in_, a.w, a.bias = N.ptr(inp), N.ptr(w), N.ptr(self.w.dev[bname])
        a.H, a.W, a.n_frames, a.frame0, a.n_out_frames = L.h, L.w, L.frames, frame0, T
        a.cin, a.cout = inp.shape[-1], w.shape[0]
        a.kt, a.kh, a.kw = kt, kh, kw
        a.res, a.out32, a.out16, a.act = N.ptr(res), N.ptr(out32), N.ptr(out16), N.ptr(act)
        a.gamma = N.ptr(self.w.dev[gamma]) if gamma else 0
        a.act_silu = silu
        a.video, a.video_channels, a.video_frame0 = N.ptr(video), video_ch, 0
        N.check(N.lib().bc_vae_conv(a, self._sp), "bc_vae_conv")
        self.launches += 1
        if self._prof is not None:
            self._mark(f"conv{kt}{kh}{kw}_{a.cin}x{a.cout}@L{lvl}",
                       2.0 * kt * kh * kw * a.cin * a.cout * L.h * L.w * T)
        if split_norm:
            N.check(N.lib().bc_vae_norm_act(N.ptr(out32), N.ptr(self.w.dev[gamma]), N.ptr(act_buf), frame0, T,
                                            L.h, L.w, w.shape[0], silu, self._sp), "bc_vae_norm_act")
            self.launches += 1
            self._mark("norm_act")

    def _scratch(self, lvl, c):
        key = (lvl, c)
        if key not in self._scr:
            self._scr[key] = self.levels[lvl].buf(self.torch, c, self.torch.float32)
        return self._scr[key]

    def _gemm(self, A, B, Cout, M, Nn, K, mode, bias=None):
        N.check(N.lib().bc_gemm_bf16(N.ptr(A), N.ptr(B), N.ptr(Cout), M, Nn, K, mode, N.ptr(bias), None,
                                     0, 1, self._sp), "bc_gemm_bf16")
        self.launches += 1

    def _resblock(self, lvl, T, n, ci, co, nxt):
        x_in, x_out = self.x[lvl][ci], self.x[lvl][co]
        res = x_in
        if ci != co:
            self._conv(lvl, T, self.raw[lvl][ci], f"{n}.sc.w", f"{n}.sc.b", 1, 1, 1, out32=x_out)
            res = x_out
        self._conv(lvl, T, self.in1[n], f"{n}.c1.w", f"{n}.c1.b", 3, 3, 3, act=self.in2[n], gamma=f"{n}.n2")
        self._conv(lvl, T, self.in2[n], f"{n}.c2.w", f"{n}.c2.b", 3, 3, 3, res=res,
                   out32=x_out if nxt.get("x", True) else None, out16=nxt.get("raw"),
                   act=nxt.get("act"), gamma=nxt.get("gamma"), silu=nxt.get("silu", 1))

    def _attention(self, lvl, T, n, c):
        L = self.levels[lvl]
        lib, sp = N.lib(), self._sp
        self._conv(lvl, T, self.attn_in, f"{n}.qkv.w", f"{n}.qkv.b", 1, 1, 1, out16=self.qkv)
        hw = L.h * L.w
        nxt = self._after[n]
        for t in range(T):
            f = 2 + t
            N.check(lib.bc_vae_attn_gather(N.ptr(self.qkv), f, L.h, L.w, c, self.np_tok, N.ptr(self.aq),
                                           N.ptr(self.ak), N.ptr(self.avt), sp), "bc_vae_attn_gather")
            self._gemm(self.aq, self.ak, self.aS, hw, self.np_tok, c, 2)
            N.check(lib.bc_vae_softmax(N.ptr(self.aS), N.ptr(self.aP), hw, self.np_tok, hw,
                                       1.0 / math.sqrt(c), sp), "bc_vae_softmax")
            self._gemm(self.aP, self.avt, self.aO, hw, c, self.np_tok, 0)
            self._gemm(self.aO, self.w.dev[f"{n}.proj.w"].reshape(c, c), self.aproj, hw, c, c, 2,
                       bias=self.w.dev[f"{n}.proj.b"])
            N.check(lib.bc_vae_attn_out(N.ptr(self.x[lvl][c]), N.ptr(self.aproj), N.ptr(self.w.dev[nxt["gamma"]]),
                                        N.ptr(nxt["act"]), f, L.h, L.w, c, sp), "bc_vae_attn_out")
            self.launches += 3
            self._mark("attention", 4.0 * hw * hw * c + 2.0 * hw * c * c)

    def _resample(self, lvl, T, n, c, kind, first):
        """Resample(up3d | up2d) of level lvl's x (c channels) -> level lvl+1;
        returns the frame count there."""
        x = self.x[lvl][c]
        fm = N.VaeFrameMap()
        frames = []
        if kind == "up3d":
            tc_in = self.raw[lvl][c]
            t0 = 1 if first else 0              # the stream's first frame is not time-upsampled ('Rep')
            if first:
                tc_in[2].zero_()                 # ... and is not part of the time conv's stream
                frames.append((0, 2, 0))
            self._conv(lvl, T - t0, tc_in, f"{n}.tc.w", f"{n}.tc.b", 3, 1, 1, frame0=2 + t0,
                       out32=self.tc_out[n])
            for t in range(t0, T):
                frames += [(1, 2 + t, 0), (1, 2 + t, c)]
        else:
            frames = [(0, 2 + t, 0) for t in range(T)]
        for j, (s, f, ch) in enumerate(frames):
            fm.src[j], fm.frame[j], fm.chan[j] = s, f, ch
        L = self.levels[lvl]
        T2 = len(frames)
        N.check(N.lib().bc_vae_upsample(N.ptr(x), N.ptr(self.tc_out.get(n)), fm, c, L.h, L.w,
                                        N.ptr(self.up_in[n]), 2, T2, self._sp), "bc_vae_upsample")
        self.launches += 1
        self._mark("upsample")
        nxt = self._after[n]
        self._conv(lvl + 1, T2, self.up_in[n], f"{n}.rs.w", f"{n}.rs.b", 1, 3, 3,
                   out32=self.x[lvl + 1][c // 2], out16=nxt.get("raw"), act=nxt.get("act"), gamma=nxt.get("gamma"))
        return T2

    def _plan_next(self):
        """For each layer: what the layer's last epilogue must produce for the
        NEXT layer (its normalised input, a raw bf16 copy, or nothing)."""
        after = {}
        seq = [("conv1", None)] + [(s[1], s) for s in self.specs] + [("head", None)]
        lvl = 0
        lvl_of = {"conv1": 0}
        for s in self.specs:
            lvl_of[s[1]] = lvl
            if s[0] in ("up3d", "up2d"):
                lvl += 1
        lvl_of["head"] = lvl
        for (name, spec), (nname, nspec) in zip(seq[:-1], seq[1:]):
            if nspec is None:                   # head
                after[name] = {"act": self.head_in, "gamma": "head.n", "x": False}
            elif nspec[0] == "res":
                d = {"act": self.in1[nname], "gamma": f"{nname}.n1"}
                if nspec[2] != nspec[3]:
                    d["raw"] = self.raw[lvl_of[nname]][nspec[2]]
                after[name] = d
            elif nspec[0] == "attn":
                after[name] = {"act": self.attn_in, "gamma": f"{nname}.norm", "silu": 0}
            elif nspec[0] == "up3d":
                after[name] = {"raw": self.raw[lvl_of[nname]][nspec[2]]}
            else:
                after[name] = {}
        return after

    def decode_block(self, z, out=None):
        """z: fp32 [T][z_dim][h][w] (device tensor or host array).  Returns
        the block's video frames [n][3][8h][8w] fp32 on the device (``out`` if
        given).  Enqueued on self.stream; the caller waits on it."""
        torch = self.torch
        cfg = self.cfg
        if not hasattr(self, "_after"):
            self._after = self._plan_next()
        if not hasattr(z, "is_cuda"):
            z = torch.from_numpy(z).to("cuda", non_blocking=True)
        T = z.shape[0]
        if tuple(z.shape[1:]) != (cfg.z_dim, cfg.latent_h, cfg.latent_w) or T != cfg.block_size:
            raise ContractViolation(f"VAE block latents {tuple(z.shape)} != "
                                    f"({cfg.block_size}, {cfg.z_dim}, {cfg.latent_h}, {cfg.latent_w})")
        first = self.first
        n_out = cfg.frames_out(T, first)
        self._sp = N.stream_ptr(self.stream)
        self.stream.wait_stream(torch.cuda.current_stream())     # z (and out) come from the caller's stream
        with torch.cuda.stream(self.stream):
            if out is None:
                out = torch.empty((n_out, 3, cfg.video_h, cfg.video_w), dtype=torch.float32, device="cuda")
            elif tuple(out.shape) != (n_out, 3, cfg.video_h, cfg.video_w):
                raise ContractViolation(f"VAE output {tuple(out.shape)} for {n_out} frames")
            z = z.float().contiguous()
            if z.device != out.device:
                raise ContractViolation("VAE latents and output on different devices")
            d = self.w.dev
            N.check(N.lib().bc_vae_prep(N.ptr(z), N.ptr(d["conv2.w"]), N.ptr(d["conv2.b"]), N.ptr(d["latent_mean"]),
                                        N.ptr(d["latent_std"]), N.ptr(self.prep), T, cfg.z_dim, cfg.latent_h,
                                        cfg.latent_w, 2, 32, self._sp), "bc_vae_prep")
            self._mark("prep")
            nxt = self._after["conv1"]
            self._conv(0, T, self.prep, "conv1.w", "conv1.b", 3, 3, 3, out32=self.x[0][self.dims[0]],
                       act=nxt["act"], gamma=nxt["gamma"])
            lvl, t = 0, T
            for s in self.specs:
                if s[0] == "res":
                    self._resblock(lvl, t, s[1], s[2], s[3], self._after[s[1]])
                elif s[0] == "attn":
                    self._attention(lvl, t, s[1], s[2])
                else:
                    t = self._resample(lvl, t, s[1], s[2], s[0], first)
                    lvl += 1
            self._conv(lvl, t, self.head_in, "head.w", "head.b", 3, 3, 3, video=out, video_ch=3)
            if t != n_out:
                raise ContractViolation(f"VAE frame count {t} != {n_out}")   # pragma: no cover
            # causal caches: the last two input frames of every kt = 3 conv
            for buf, l in self.hist:
                tl = self._frames_at(l, T, first)
                buf[0:2].copy_(buf[tl:tl + 2])
            self.launches += 2
            self._mark("cache_copies")
        self.first = False
        return out

    def wait(self, stream=None):
        """Make `stream` (default: the current stream) wait for every decode
        enqueued so far -- before reading a returned video tensor."""
        torch = self.torch
        (stream or torch.cuda.current_stream()).wait_stream(self.stream)

    def _frames_at(self, lvl, T, first):
        t = T
        k = 0
        for s in self.specs:
            if k == lvl:
                break
            if s[0] == "up3d":
                t = 1 + 2 * (t - 1) if first else 2 * t
                k += 1
            elif s[0] == "up2d":
                k += 1
        return t

    def flops_per_block(self, first: bool = False) -> float:
        """Algorithmic FLOPs of one block's decode (convs as 2*taps*cin*cout
        per output pixel, attention 4*(hw)^2*c per frame)."""
        cfg = self.cfg
        T = cfg.block_size
        tot = 0.0
        L0 = self.levels[0]
        hw = L0.h * L0.w
        tot += 2 * 27 * cfg.z_dim * self.dims[0] * hw * T
        lvl, t = 0, T
        for s in self.specs:
            hw = self.levels[lvl].h * self.levels[lvl].w
            if s[0] == "res":
                _, _, ci, co = s
                tot += 2 * 27 * (ci * co + co * co) * hw * t + (2 * ci * co * hw * t if ci != co else 0)
            elif s[0] == "attn":
                c = s[2]
                tot += (2 * c * 3 * c * hw + 4 * hw * hw * c + 2 * c * c * hw) * t
            else:
                c = s[2]
                t0 = 1 if first else 0
                if s[0] == "up3d":
                    tot += 2 * 3 * c * 2 * c * hw * (t - t0)
                    t = 1 + 2 * (t - 1) if first else 2 * t
                lvl += 1
                tot += 2 * 9 * c * (c // 2) * self.levels[lvl].h * self.levels[lvl].w * t
        hw = self.levels[lvl].h * self.levels[lvl].w
        tot += 2 * 27 * self.last * 3 * hw * t
        return tot
