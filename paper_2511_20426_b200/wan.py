"""Wan2.1-shaped model family on the device (configs 2-5).

``WanWeights`` holds random-init weights of the Wan2.1 T2V architecture
(patch embed (1,2,2) -> d, text MLP 4096 -> d, time
MLP 256 -> d -> 6d, L blocks of {AdaLN self-attention with q/k RMSNorm and
3-D RoPE, affine-LN cross-attention over 512 text tokens, AdaLN GELU FFN},
head LN + modulation -> 64 -> unpatchify) as caller-owned torch tensors:
linear weights bf16 [out][in], vectors fp32.  ``WanRuntime`` binds them to
the C-ABI context (``bc_wan_create``) and runs one cascade iteration per
``bc_wan_step`` call; ``WanSession`` is the engine-facing session that keeps
latents and the KV arena resident on the device.

Noise parameterisation is the reference's (sigma = level / 1000, no shift;
SPEC.md:104, denoiser.py:367); the head predicts flow v and the fused
update computes x0 = x_t - sigma * v before renoising.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import _native as N
from .errors import ContractViolation, InvalidInputError, NumericError
from .kvpool import SlotAllocator, SlotKV

POST_RENOISE, POST_EMIT, POST_CACHE, POST_X0 = 0, 1, 2, 3

_VECTOR_FIELDS = {"patch_b", "text_b1", "text_b2", "time_b1", "time_b2", "tproj_b", "head_b",
                  "head_mod", "qkv_b", "o_b", "cq_b", "ckv_b", "co_b", "ffn1_b", "ffn2_b",
                  "norm_q", "norm_k", "cnorm_q", "cnorm_k", "norm3_w", "norm3_b", "modulation"}


def param_shapes(cfg) -> dict:
    """name -> (shape, fan_in or None, kind).  kind: 'w' linear weight,
    'b' bias, 'one' norm weight around 1, 'mod' modulation table."""
    d, L, ffn = cfg.model_dim, cfg.layers, cfg.ffn_dim
    return {
        "patch_w": ((d, 64), 64, "w"), "patch_b": ((d,), None, "b"),
        "text_w1": ((d, cfg.text_dim), cfg.text_dim, "w"), "text_b1": ((d,), None, "b"),
        "text_w2": ((d, d), d, "w"), "text_b2": ((d,), None, "b"),
        "time_w1": ((d, cfg.freq_dim), cfg.freq_dim, "w"), "time_b1": ((d,), None, "b"),
        "time_w2": ((d, d), d, "w"), "time_b2": ((d,), None, "b"),
        "tproj_w": ((6 * d, d), d, "w"), "tproj_b": ((6 * d,), None, "b"),
        "head_w": ((64, d), d, "w"), "head_b": ((64,), None, "b"),
        "head_mod": ((2, d), None, "mod"),
        "qkv_w": ((L, 3 * d, d), d, "w"), "qkv_b": ((L, 3 * d), None, "b"),
        "o_w": ((L, d, d), d, "w"), "o_b": ((L, d), None, "b"),
        "cq_w": ((L, d, d), d, "w"), "cq_b": ((L, d), None, "b"),
        "ckv_w": ((L, 2 * d, d), d, "w"), "ckv_b": ((L, 2 * d), None, "b"),
        "co_w": ((L, d, d), d, "w"), "co_b": ((L, d), None, "b"),
        "ffn1_w": ((L, ffn, d), d, "w"), "ffn1_b": ((L, ffn), None, "b"),
        "ffn2_w": ((L, d, ffn), ffn, "w"), "ffn2_b": ((L, d), None, "b"),
        "norm_q": ((L, d), None, "one"), "norm_k": ((L, d), None, "one"),
        "cnorm_q": ((L, d), None, "one"), "cnorm_k": ((L, d), None, "one"),
        "norm3_w": ((L, d), None, "one"), "norm3_b": ((L, d), None, "b"),
        "modulation": ((L, 6, d), None, "mod"),
    }


class WanWeights:
    """Random-init Wan2.1-shaped weights, resident on the device."""

    def __init__(self, config, tensors: dict, seed: int):
        self.config = config
        self.t = tensors
        self.seed = seed
        self.layers = config.layers
        self.heads = config.heads
        self._runtime = None

    @classmethod
    def random(cls, config, seed: int = 7) -> "WanWeights":
        torch = N.torch_mod()
        gen = torch.Generator(device="cuda")
        gen.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
        d = config.model_dim
        out = {}
        for name, (shape, fan_in, kind) in param_shapes(config).items():
            if kind == "w":
                t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
                rows = t.view(-1, shape[-1])
                step = max(1, (1 << 26) // shape[-1])          # bounded fp32 temporaries
                for r0 in range(0, rows.shape[0], step):
                    chunk = torch.randn((min(step, rows.shape[0] - r0), shape[-1]),
                                        generator=gen, device="cuda")
                    rows[r0:r0 + chunk.shape[0]] = (chunk / math.sqrt(fan_in)).bfloat16()
            else:
                r = torch.randn(shape, generator=gen, device="cuda")
                if kind == "b":
                    t = 0.02 * r
                elif kind == "one":
                    t = 1.0 + 0.05 * r
                else:
                    t = r / math.sqrt(d)
                t = t.float().contiguous()
            out[name] = t
        return cls(config, out, seed)

    def host_params(self) -> dict:
        """fp32 numpy copies (bf16 values upcast) -- for the CPU oracle."""
        return {k: v.float().cpu().numpy() for k, v in self.t.items()}

    def nbytes(self) -> int:
        return sum(v.numel() * v.element_size() for v in self.t.values())

    def runtime(self) -> "WanRuntime":
        if self._runtime is None:
            self._runtime = WanRuntime(self)
        return self._runtime


def text_states(cond, text_len: int, text_dim: int) -> np.ndarray:
    """Synthetic text-encoder states for a prompt: row r is
    standard_normal(text_dim) from Philox(key = sha256(prompt)[:16] as two
    uint64, counter = [r, 1, 0, 0]).  float32 [text_len][text_dim]."""
    if hasattr(cond, "key_words"):
        key = cond.key_words()
    else:   # the reference's Conditioning (core.py:131-141) keeps the prompt, not the digest
        import hashlib
        key = np.frombuffer(hashlib.sha256(cond.prompt.encode("utf-8")).digest()[:16], dtype=np.uint64)
    out = np.empty((text_len, text_dim), dtype=np.float32)
    N.run_noise_tasks([(int(key[0]), int(key[1]), (r, 1, 0, 0), out[r]) for r in range(text_len)], 1)
    return out


class _Ctx:
    """One bc_wan_ctx plus the arena / workspace it was created over."""

    def __init__(self, weights: WanWeights, max_entries: int, n_slots: int, arena=None):
        torch = N.torch_mod()
        cfg = weights.config
        self.cfg, self.weights = cfg, weights
        self.T = cfg.tokens_per_block
        self.d = cfg.model_dim
        self.n_slots, self.max_entries = n_slots, max_entries
        dims = N.WanDims(layers=cfg.layers, heads=cfg.heads, head_dim=cfg.head_dim,
                         ffn_dim=cfg.ffn_dim, text_len=cfg.text_len, text_dim=cfg.text_dim,
                         freq_dim=cfg.freq_dim, latent_h=cfg.latent_height,
                         latent_w=cfg.latent_width, block_size=cfg.block_size,
                         n_slots=n_slots, max_entries=max_entries)
        self.dims = dims
        need = N.lib().bc_wan_workspace_bytes(dims)
        if need < 0:
            raise ContractViolation("bc_wan_workspace_bytes rejected the dims")
        # no zero fill (11-54 GB): a slot is always written (its block's K/V
        # in layer part A) before any attention reads it, and key rows past a
        # slot's end are TMA out-of-bounds zero fill
        self.arena = arena if arena is not None else torch.empty(
            (cfg.layers, n_slots, 2, self.T, self.d), dtype=torch.bfloat16, device="cuda")
        self.workspace = torch.empty(int(need), dtype=torch.uint8, device="cuda")
        prm = N.WanParams()
        for name in N.WAN_PARAM_FIELDS:
            setattr(prm, name, N.ptr(weights.t[name]))
        self.params = prm
        h = ctypes.c_void_p()
        N.check(N.lib().bc_wan_create(dims, prm, N.ptr(self.arena), N.ptr(self.workspace),
                                      int(need), ctypes.byref(h)), "bc_wan_create")
        self.handle = h
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.text_id = None

    def set_text(self, cond):
        if self.text_id == cond.id:
            return
        torch = N.torch_mod()
        cfg = self.cfg
        host = torch.from_numpy(text_states(cond, cfg.text_len, cfg.text_dim))
        dev = host.pin_memory().cuda(non_blocking=True)
        N.check(N.lib().bc_wan_set_text(self.handle, N.ptr(dev), N.stream_ptr()), "bc_wan_set_text")
        self._text_keep = dev
        self.text_id = cond.id

    def step(self, batch, upd):
        N.check(N.lib().bc_wan_step(self.handle, batch, upd, N.ptr(self.status), N.stream_ptr()),
                "bc_wan_step")

    def check_status(self):
        code = int(self.status.item())
        if code:
            self.status.zero_()
            err = NumericError(f"non-finite latents in block {code - 1}")
            err.block_index = code - 1
            raise err

    def read_kv(self, slot, layer, which):
        if self.arena is None:
            raise ContractViolation("KV of a closed session is no longer resident")
        arr = self.arena[layer, slot, which].float().cpu().numpy()
        return arr.reshape(self.T, self.cfg.heads, self.cfg.head_dim)

    @property
    def layers(self):
        return self.cfg.layers

    def read(self, slot, layer, which):
        return self.read_kv(slot, layer, which)

    def close(self):
        """Destroy the C context and drop the device buffers (results that
        still reference this context, e.g. a RunResult's pool handles, no
        longer pin ~11-54 GB of KV arena)."""
        if self.handle:
            N.lib().bc_wan_destroy(self.handle)
            self.handle = None
        self.arena = None
        self.workspace = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _make_update(posts, latents, eps, outs, next_levels):
    u = N.WanUpdate()
    for i, kind in enumerate(posts):
        u.post[i] = kind
        u.next_level[i] = float(next_levels[i]) if next_levels[i] is not None else 0.0
        u.latents[i] = N.ptr(latents[i])
        u.eps[i] = N.ptr(eps[i]) if eps[i] is not None else None
        u.out[i] = N.ptr(outs[i]) if outs[i] is not None else None
    return u


class _Lease:
    """A session's view of a (pooled) context for the pool's KV handles:
    revoked when the session closes, so a finished run's handles can never
    read a later session's KV out of a reused arena."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.layers = ctx.layers

    def read(self, slot, layer, which):
        if self.ctx is None:
            raise ContractViolation("KV of a closed session is no longer resident")
        return self.ctx.read_kv(slot, layer, which)


class _OpSlot:
    """What an operator-path K/V handle reads through: one slot of the
    runtime's operator arena at the generation the handle was made in."""

    def __init__(self, op, slot, gen):
        self.op, self.slot, self.gen = op, slot, gen
        self.layers = op.ctx.layers

    def valid(self):
        return self.op.ctx.handle is not None and self.op.gen[self.slot] == self.gen

    def read(self, slot, layer, which):
        if not self.valid():
            raise ContractViolation("K/V handle of a recycled operator slot (the block left the "
                                    "arena); keep its host arrays if it is needed later")
        return self.op.ctx.read_kv(slot, layer, which)


class _OpArena:
    """Slot bookkeeping of the operator path: generation per slot and a
    least-recently-used choice of the slot a new block overwrites (never one
    the current call attends to)."""

    def __init__(self, ctx):
        self.ctx = ctx
        self.gen = [0] * ctx.n_slots
        self.used = [0] * ctx.n_slots   # call counter of the last use
        self.calls = 0
        self.uploads = 0                # pool blocks that had to come from host arrays

    def resident_slot(self, kv):
        """The slot of a still-valid handle of THIS arena, else None.  ``kv``
        is a SlotKV or any sequence of its per-layer views (the reference
        KVPool stores ``tuple(kv_layers)``, kvpool.py:51-53)."""
        ref = getattr(kv, "arena", None)
        if ref is None and len(kv) and all(getattr(l, "_arena", None) is getattr(kv[0], "_arena", 0) for l in kv):
            ref = getattr(kv[0], "_arena", None)
        if isinstance(ref, _OpSlot) and ref.op is self and ref.valid():
            self.used[ref.slot] = self.calls + 1
            return ref.slot
        return None

    def take(self, pinned, block):
        self.calls += 1
        free = [s for s in range(self.ctx.n_slots) if s not in pinned]
        if not free:
            raise ContractViolation("operator arena exhausted")
        s = min(free, key=lambda x: self.used[x])
        self.gen[s] += 1               # whatever the slot held is gone
        self.used[s] = self.calls
        return s

    def ref(self, slot):
        return _OpSlot(self, slot, self.gen[slot])

    def close(self):
        self.ctx.close()


class WanRuntime:
    def __init__(self, weights: WanWeights):
        self.weights = weights
        self.cfg = weights.config
        self._cached = None   # (key, _Ctx) kept between sessions (arena, workspace, text K/V)

    def acquire_ctx(self, width, n_slots):
        """A context for a session: the cached one when the geometry matches
        (no allocation / arena setup / text re-projection for a repeated
        prompt), else a new one."""
        key = (width, n_slots)
        if self._cached is not None:
            ck, ctx = self._cached
            self._cached = None
            if ck == key:
                return ctx
            ctx.close()
        return _Ctx(self.weights, width, n_slots)

    def release_ctx(self, ctx):
        N.torch_mod().cuda.current_stream().synchronize()
        if self._cached is not None:
            self._cached[1].close()
        self._cached = ((ctx.max_entries, ctx.n_slots), ctx)

    def release_cached(self):
        """Free the cached contexts' device memory (KV arena + workspace) of
        the session path and of the operator path."""
        if self._cached is not None:
            self._cached[1].close()
            self._cached = None
        if getattr(self, "_op", None) is not None:
            self._op.close()
            self._op = None

    # reference operator contract (denoiser.forward) ----------------------
    def forward(self, batch, pool_kv, mask):
        """``denoiser.forward`` for Wan weights (reference ``denoiser.py:299-357``
        contract).  The operator path keeps one persistent context (arena,
        workspace, text K/V of the last conditioning) in the runtime, and
        returns every entry's fresh K/V as a device-resident handle
        (:class:`~.kvpool.SlotKV` over :class:`_OpSlot`): when the caller --
        e.g. the reference engine's ``apply_results`` / ``KVPool`` -- hands
        those handles back as pool KV, the blocks are attended in place (no
        host round trip of ~0.9 GB per block at 1.3B).  Host-array LayerKV
        (any other producer) is uploaded into a free slot.  A slot that is
        recycled bumps its generation, so a stale handle raises instead of
        reading another block's K/V."""
        from .denoiser import EntryOutput, visible_block_lists
        from .kvpool import SlotKV
        torch = N.torch_mod()
        cfg = self.cfg
        S, C, H, W = cfg.block_size, cfg.latent_channels, cfg.latent_height, cfg.latent_width
        if len({e.conditioning.id for e in batch}) != 1:
            raise ContractViolation("the Wan forward takes one conditioning per call")
        pool_blocks = list(mask.pool_blocks)
        blocks = [e.block_index for e in batch]
        op = self._op_arena(len(batch), len(pool_blocks) + len(blocks))
        slot_of = {}
        for b in pool_blocks:                   # resident handles first: they pin their slots
            s_ = op.resident_slot(pool_kv[b])
            if s_ is not None:
                slot_of[b] = s_
        pinned = set(slot_of.values())
        for b in pool_blocks:
            if b not in slot_of:                # host arrays (or a foreign / stale handle): upload
                slot_of[b] = op.take(pinned, b)
                pinned.add(slot_of[b])
                op.uploads += 1
                for layer, kv in enumerate(pool_kv[b]):
                    for which, arr in ((0, kv.keys), (1, kv.values)):
                        op.ctx.arena[layer, slot_of[b], which].copy_(
                            torch.as_tensor(np.asarray(arr, dtype=np.float32)).reshape(op.ctx.T, op.ctx.d))
        for b in blocks:                        # each entry's fresh K/V goes to a slot of its own
            slot_of[b] = op.take(pinned, b)
            pinned.add(slot_of[b])
        op.ctx.set_text(batch[0].conditioning)
        host = [not hasattr(e.latents, "is_cuda") for e in batch]
        lat = [torch.as_tensor(np.asarray(e.latents, dtype=np.float32)).cuda() if h
               else e.latents.float() for e, h in zip(batch, host)]
        lat = [x.reshape(S, C, H, W).contiguous().clone() for x in lat]
        outs = [torch.empty_like(x) for x in lat]
        vis = [[slot_of[v] for v in lst] for lst in visible_block_lists(mask)]
        bt = N.make_batch(S, blocks, [e.noise_level for e in batch], [slot_of[b] for b in blocks], vis)
        upd = _make_update([POST_X0] * len(batch), lat, [None] * len(batch), outs, [None] * len(batch))
        op.ctx.step(bt, upd)
        torch.cuda.current_stream().synchronize()
        op.ctx.check_status()
        results = []
        for i, e in enumerate(batch):
            x0 = outs[i].reshape(S, -1)
            x0 = x0.cpu().numpy().astype(np.float64) if host[i] else x0
            kv = SlotKV(op.ref(slot_of[e.block_index]), slot_of[e.block_index], e.block_index,
                        e.noise_level, e.conditioning.id, S)
            results.append(EntryOutput(block_index=e.block_index, x0=x0, kv=kv))
        return results

    def _op_arena(self, entries, slots_needed):
        """The operator path's persistent context, grown when a call needs
        more entries or slots than it has (the default fits the config's
        cascade: W + sink + width + 1 slots)."""
        cfg = self.cfg
        op = getattr(self, "_op", None)
        if op is None or op.ctx.max_entries < entries or op.ctx.n_slots < slots_needed:
            if op is not None:
                op.close()
            width = max(entries, min(cfg.cascade_width, cfg.num_blocks))
            n_slots = max(slots_needed, cfg.window_blocks + cfg.sink_blocks + width + 1)
            op = self._op = _OpArena(_Ctx(self.weights, width, n_slots))
        return op

    def open_session(self, config, conditioning, session_seed, noise_feed=None):
        from . import distributed
        try:
            multi = distributed.dit_world() > 1
        except ImportError:  # pragma: no cover
            multi = False
        if multi:
            return distributed.DistWanSession(self, config, conditioning, session_seed, noise_feed)
        if distributed.EMULATE and config.workers > 1:
            return distributed.EmulatedRanks(self, config, conditioning, session_seed,
                                             config.workers, noise_feed)
        return WanSession(self, config, conditioning, session_seed, noise_feed)


class HostNoiseFeed:
    """Counter-keyed noise for the device: generated on the host by the
    native numpy-exact generator into pinned buffers, copied H2D on the
    launching stream (a ring of pinned buffers guarded by events)."""

    def __init__(self, session_seed, cfg, ring: int = 24):
        torch = N.torch_mod()
        from .core import NoiseStream
        self.stream = NoiseStream(session_seed, cfg.latent_dim)
        self.shape = (cfg.block_size, cfg.latent_channels, cfg.latent_height, cfg.latent_width)
        self.S = cfg.block_size
        self.ring = [torch.empty(self.shape, dtype=torch.float32, pin_memory=True) for _ in range(ring)]
        self.events = [None] * ring
        self.next = 0
        self.h2d_bytes = 0
        # host threads for the generator: the node's cores shared by the ranks
        # on it (every rank of the rows partition draws every entry's noise)
        env = os.environ.get("BC_NOISE_THREADS")
        local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
        self.threads = int(env) if env else max(1, (os.cpu_count() or 1) // local)

    def fetch(self, requests, dests):
        """requests: [(block, pass)], dests: device tensors of self.shape.
        A key requested for several destinations (per-rank replicas) is
        generated once; more keys than ring buffers go in chunks."""
        torch = N.torch_mod()
        uniq = list(dict.fromkeys(requests))
        for c0 in range(0, len(uniq), len(self.ring)):
            chunk = uniq[c0:c0 + len(self.ring)]
            bufs = []
            for _ in chunk:
                i = self.next
                self.next = (self.next + 1) % len(self.ring)
                if self.events[i] is not None:
                    self.events[i].synchronize()
                bufs.append(i)
            tasks = []
            for (block, pass_index), i in zip(chunk, bufs):
                host = self.ring[i].numpy().reshape(self.S, -1)
                tasks += [(self.stream.session_seed, 0, (block, pass_index, block * self.S + f, 0), host[f])
                          for f in range(self.S)]
            N.run_noise_tasks(tasks, 1, self.threads)
            for key, i in zip(chunk, bufs):
                for k, dst in zip(requests, dests):
                    if k == key:
                        dst.copy_(self.ring[i], non_blocking=True)
                        self.h2d_bytes += dst.numel() * 4
                ev = torch.cuda.Event()
                ev.record()
                self.events[i] = ev


class ResidentNoiseFeed:
    """All noise of a run pre-generated into device memory (for the
    device-resident `value` measurement: inputs already in HBM)."""

    def __init__(self, session_seed, cfg, keys):
        torch = N.torch_mod()
        host = HostNoiseFeed(session_seed, cfg, ring=4)
        self.table = {}
        for k in keys:
            t = torch.empty(host.shape, dtype=torch.float32, device="cuda")
            host.fetch([k], [t])
            self.table[k] = t
        torch.cuda.synchronize()
        self.h2d_bytes = 0

    def fetch(self, requests, dests):
        for k, dst in zip(requests, dests):
            dst.copy_(self.table[k])


def run_noise_keys(cfg, offset=None):
    """Every (block, pass) noise key a run consumes: pass 0 initial latents
    and passes 1..emit for renoise (reference scheduler.py:216-220)."""
    emit = len(cfg.denoise_levels) - 1
    return [(b, p) for b in range(cfg.num_blocks) for p in range(0, emit + 1)]


class WanSession:
    """Engine session: device-resident latents, KV arena and outputs."""

    def __init__(self, rt: WanRuntime, config, conditioning, session_seed, noise_feed=None):
        torch = N.torch_mod()
        self.torch = torch
        self.rt, self.cfg = rt, config
        width = min(config.cascade_width, config.num_blocks)
        self.ctx = rt.acquire_ctx(width, config.window_blocks + config.sink_blocks + width + 1)
        self.lease = _Lease(self.ctx)
        self.slots = SlotAllocator(self.ctx.n_slots)
        self.shape = (config.block_size, config.latent_channels, config.latent_height,
                      config.latent_width)
        self.noise = noise_feed if noise_feed is not None else HostNoiseFeed(session_seed, config)
        self.latents, self.final, self.tags = {}, {}, {}
        self.host_out = {}
        # emitted blocks whose D2H copy is in flight (event) / already
        # converted to the API's float64 arrays while the device kept working
        self.host_pending, self.host_f64 = {}, {}
        # one pinned staging area for every emitted block (no per-emission
        # cudaHostAlloc, which would serialise against the device)
        self.host_buf = torch.empty((config.num_blocks,) + tuple(self.shape),
                                    dtype=torch.float32, pin_memory=True)
        self.eps = [torch.empty(self.shape, dtype=torch.float32, device="cuda")
                    for _ in range(width)]
        self.events = []
        self.stalls = {}
        self.d2h_bytes = 0
        self.set_conditioning(conditioning)
        self._mark()

    def _mark(self):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append(ev)

    def set_conditioning(self, cond):
        self.cond = cond
        self.ctx.set_text(cond)

    def _convert_landed(self):
        # host-side float64 conversion of blocks whose D2H copy has landed,
        # done while the device runs (not all at the end of the run)
        for b, ev in list(self.host_pending.items()):
            if ev.query():
                self.host_f64[b] = self.host_out[b].numpy().reshape(self.cfg.block_size, -1).astype(np.float64)
                del self.host_pending[b]

    def step(self, plan, mask, pool, vis_lists, posts):
        torch = self.torch
        self._convert_landed()
        init_req, init_dst = [], []
        for e in plan.entries:
            self.slots.acquire(e.block_index)
            if e.pass_index == 0 and e.block_index not in self.latents:
                t = torch.empty(self.shape, dtype=torch.float32, device="cuda")
                self.latents[e.block_index] = t
                init_req.append((e.block_index, 0))
                init_dst.append(t)
        eps_req, eps_dst, eps_ptrs, outs, next_levels = [], [], [], [], []
        for i, (e, (kind, next_pass, next_level)) in enumerate(zip(plan.entries, posts)):
            if kind == POST_RENOISE:
                eps_req.append((e.block_index, next_pass))
                eps_dst.append(self.eps[i])
                eps_ptrs.append(self.eps[i])
            else:
                eps_ptrs.append(None)
            if kind == POST_EMIT:
                out = torch.empty(self.shape, dtype=torch.float32, device="cuda")
                self.final[e.block_index] = out
                outs.append(out)
            else:
                outs.append(None)
            next_levels.append(next_level)
        if init_req or eps_req:
            self.noise.fetch(init_req + eps_req, init_dst + eps_dst)
        vis = [[self.slots.slot_of(v) for v in lst] for lst in vis_lists]
        blocks = plan.blocks
        bt = N.make_batch(self.cfg.block_size, blocks, [e.noise_level for e in plan.entries],
                          [self.slots.slot_of(b) for b in blocks], vis)
        upd = _make_update([p[0] for p in posts], [self.latents[b] for b in blocks], eps_ptrs,
                           outs, next_levels)
        self.ctx.step(bt, upd)
        for e, (kind, _, _) in zip(plan.entries, posts):
            self.tags[e.block_index] = (e.noise_level, self.cond.id)
            if kind == POST_EMIT:
                host = self.host_buf[e.block_index]
                host.copy_(self.final[e.block_index], non_blocking=True)
                self.host_out[e.block_index] = host
                self.host_f64.pop(e.block_index, None)
                ev = torch.cuda.Event()
                ev.record()
                self.host_pending[e.block_index] = ev
                self.d2h_bytes += host.numel() * 4
            elif kind == POST_CACHE:
                self.latents.pop(e.block_index, None)
        self._mark()

    def recache_block(self, block, mask, vis_list):
        """One causal level-0 forward of an emitted block from its x0 under
        the current conditioning, rewriting its KV slot in place (recache
        baseline, reference kvpool.py:109-140; not the product switch)."""
        vis = [self.slots.slot_of(v) for v in vis_list]
        bt = N.make_batch(self.cfg.block_size, [block], [0.0], [self.slots.slot_of(block)], [vis])
        upd = _make_update([POST_CACHE], [self.final[block]], [None], [None], [None])
        self.ctx.step(bt, upd)
        self.tags[block] = (0.0, self.cond.id)

    def begin_stall(self):
        self._stall0 = self.torch.cuda.Event(enable_timing=True)
        self._stall0.record()

    def end_stall(self, iteration):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        self.stalls[iteration] = (self._stall0, ev)

    def stall_seconds(self):
        self.torch.cuda.current_stream().synchronize()
        return {i: a.elapsed_time(b) / 1e3 for i, (a, b) in self.stalls.items()}

    def kv_handle(self, block):
        level, cid = self.tags[block]
        return SlotKV(self.lease, self.slots.slot_of(block), block, level, cid, self.cfg.block_size)

    def release(self, block):
        self.slots.release(block)

    def emitted_host(self, block):
        self.torch.cuda.current_stream().synchronize()
        self.ctx.check_status()
        self.host_pending.pop(block, None)
        cached = self.host_f64.pop(block, None)
        if cached is not None:
            return cached
        return self.host_out[block].numpy().reshape(self.cfg.block_size, -1).astype(np.float64)

    def emitted_device(self, block):
        return self.final[block]

    def release_device(self):
        self.torch.cuda.current_stream().synchronize()
        if self.lease.ctx is not None:
            self.lease.ctx = None
            self.rt.release_ctx(self.ctx)
        self.latents.clear()
        self.final.clear()

    def fill_wall_times(self, events):
        if not events:
            return
        self.torch.cuda.current_stream().synchronize()
        self.ctx.check_status()
        first = self.events[0]
        for ev in events:
            t0, t1 = self.events[ev.iteration], self.events[ev.iteration + 1]
            ev.wall_seconds = t0.elapsed_time(t1) / 1e3
            ev.wall_clock = first.elapsed_time(t1) / 1e3
            if ev.iteration in self.stalls:  # on the clock, not in the iteration
                s0, s1 = self.stalls[ev.iteration]
                ev.wall_seconds -= s0.elapsed_time(s1) / 1e3

    def close(self):
        self.release_device()
