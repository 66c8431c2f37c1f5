"""Device runtime for the reference's toy DiT (config 1), float64 on the GPU.

Wraps ``bc_toy_forward`` / ``bc_renoise_f64`` (csrc/toy.cu).  Two entry
points share the kernels:

* :meth:`ToyRuntime.forward` -- the reference operator contract
  (``denoiser.forward``): host arrays in, host arrays out, pool KV uploaded
  into a scratch arena per call;
* :meth:`ToyRuntime.open_session` -- what the engine uses: latents, KV
  arena and emitted blocks stay resident on the device for the whole run.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _native as N
from .core import NoiseStream
from .errors import ContractViolation, NumericError
from .kvpool import SlotAllocator, SlotKV

_RUNTIMES = weakref.WeakKeyDictionary()


def toy_runtime(weights) -> "ToyRuntime":
    rt = _RUNTIMES.get(weights)
    if rt is None:
        rt = ToyRuntime(weights)
        _RUNTIMES[weights] = rt
    return rt


class _Arena:
    """[layers][n_slots][2][S][D] float64 device arena."""

    def __init__(self, torch, layers, n_slots, S, D, heads):
        self.layers, self.n_slots, self.S, self.D, self.heads = layers, n_slots, S, D, heads
        self.buf = torch.zeros((layers, n_slots, 2, S, D), dtype=torch.float64, device="cuda")

    def read(self, slot, layer, which):
        arr = self.buf[layer, slot, which].cpu().numpy()
        return arr.reshape(self.S, self.heads, self.D // self.heads)

    def write(self, slot, layer, which, host):
        import torch
        self.buf[layer, slot, which].copy_(
            torch.from_numpy(np.ascontiguousarray(host, dtype=np.float64).reshape(self.S, self.D)))


class ToyRuntime:
    def __init__(self, weights):
        torch = N.torch_mod()
        self.torch = torch
        self.weights = weights
        self.L, self.H, self.D, self.Dc = weights.layers, weights.heads, weights.latent_dim, weights.cond_dim
        self._dev = {name: torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).cuda()
                     for name, arr in zip(("w_in", "w_cond", "w_level", "w_q", "w_k", "w_v",
                                           "w_o", "w_head"), weights.arrays())}
        w = N.ToyWeights()
        for name, t in self._dev.items():
            setattr(w, name, N.ptr(t))
        w.layers, w.heads, w.dim, w.cond_dim = self.L, self.H, self.D, self.Dc
        self._w = w
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")

    # shared launch --------------------------------------------------------
    def launch(self, batch, latents, conds, arena, x0s, workspace):
        n = batch.n_entries
        lat = (C_void_p_array(n))(*[N.ptr(t) for t in latents])
        cnd = (C_void_p_array(n))(*[N.ptr(t) for t in conds])
        out = (C_void_p_array(n))(*[N.ptr(t) for t in x0s])
        N.check(N.lib().bc_toy_forward(self._w, batch, lat, cnd, N.ptr(arena.buf),
                                       arena.n_slots, out, N.ptr(workspace),
                                       N.ptr(self.status), N.stream_ptr()),
                "bc_toy_forward")

    def check_status(self):
        code = int(self.status.item())
        if code:
            self.status.zero_()
            err = NumericError(f"non-finite latents in block {code - 1}")
            err.block_index = code - 1
            raise err

    # reference operator contract ---------------------------------------
    def forward(self, batch, pool_kv, mask):
        from .denoiser import EntryOutput, LayerKV, visible_block_lists
        torch = self.torch
        S = mask.block_size
        pool_blocks = list(mask.pool_blocks)
        blocks = [e.block_index for e in batch]
        slot_of = {b: i for i, b in enumerate(pool_blocks + blocks)}
        arena = _Arena(torch, self.L, len(slot_of), S, self.D, self.H)
        for b in pool_blocks:
            for layer, kv in enumerate(pool_kv[b]):
                arena.write(slot_of[b], layer, 0, kv.keys)
                arena.write(slot_of[b], layer, 1, kv.values)
        host = [not hasattr(e.latents, "is_cuda") for e in batch]
        lat = [torch.from_numpy(np.ascontiguousarray(e.latents, dtype=np.float64)).cuda()
               if h else e.latents.to(torch.float64).contiguous() for e, h in zip(batch, host)]
        conds = [torch.from_numpy(np.array(e.conditioning.embedding, dtype=np.float64)).cuda()
                 for e in batch]
        x0s = [torch.empty((S, self.D), dtype=torch.float64, device="cuda") for _ in batch]
        ws = torch.empty(2 * len(batch) * S * self.D, dtype=torch.float64, device="cuda")
        vis = [[slot_of[v] for v in lst] for lst in visible_block_lists(mask)]
        bt = N.make_batch(S, blocks, [e.noise_level for e in batch],
                          [slot_of[b] for b in blocks], vis)
        self.launch(bt, lat, conds, arena, x0s, ws)
        torch.cuda.current_stream().synchronize()
        self.check_status()
        outs = []
        for i, e in enumerate(batch):
            kv = tuple(LayerKV(block_index=e.block_index, layer_index=l,
                               keys=arena.read(slot_of[e.block_index], l, 0),
                               values=arena.read(slot_of[e.block_index], l, 1),
                               noise_tag=e.noise_level, conditioning_id=e.conditioning.id)
                       for l in range(self.L))
            x0 = x0s[i].cpu().numpy() if host[i] else x0s[i]
            outs.append(EntryOutput(block_index=e.block_index, x0=x0, kv=kv))
        return outs

    # engine session ------------------------------------------------------
    def open_session(self, config, conditioning, session_seed, noise_feed=None):
        return ToySession(self, config, conditioning, session_seed)


def C_void_p_array(n):
    import ctypes
    return ctypes.c_void_p * n


class ToySession:
    def __init__(self, rt: ToyRuntime, config, conditioning, session_seed):
        torch = rt.torch
        self.rt, self.torch = rt, torch
        self.S = config.block_size
        self.D = rt.D
        width = min(config.cascade_width, config.num_blocks)
        self.arena = _Arena(torch, rt.L, config.window_blocks + config.sink_blocks + width + 1,
                            self.S, self.D, rt.H)
        self.slots = SlotAllocator(self.arena.n_slots)
        self.noise = NoiseStream(session_seed, config.latent_dim)
        self.latents = {}
        self.final = {}
        self.tags = {}
        self.ws = torch.empty(2 * N.MAX_ENTRIES * self.S * self.D, dtype=torch.float64,
                              device="cuda")
        self.x0 = [torch.empty((self.S, self.D), dtype=torch.float64, device="cuda")
                   for _ in range(N.MAX_ENTRIES)]
        self.events = []
        self.stalls = {}
        self._staged = []
        self.set_conditioning(conditioning)
        self._mark()

    def _mark(self):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append(ev)

    def _upload_noise(self, block, pass_index):
        # pinned staging + asynchronous copy: a pageable .cuda() waits for the
        # whole queue and made the host loop wait on the device every draw
        host = self.torch.from_numpy(self.noise.block_noise(block, pass_index, block * self.S, self.S))
        pinned = host.pin_memory()
        self._staged.append(pinned)   # alive until the session ends
        return pinned.cuda(non_blocking=True)

    def set_conditioning(self, cond):
        self.cond = cond
        self.cond_dev = self.torch.from_numpy(np.array(cond.embedding, dtype=np.float64)).cuda()

    def step(self, plan, mask, pool, vis_lists, posts):
        from .engine import POST_CACHE, POST_EMIT, POST_RENOISE
        rt = self.rt
        blocks = plan.blocks
        for e in plan.entries:
            self.slots.acquire(e.block_index)
            if e.pass_index == 0 and e.block_index not in self.latents:
                self.latents[e.block_index] = self._upload_noise(e.block_index, 0)
        vis = [[self.slots.slot_of(v) for v in lst] for lst in vis_lists]
        bt = N.make_batch(self.S, blocks, [e.noise_level for e in plan.entries],
                          [self.slots.slot_of(b) for b in blocks], vis)
        x0s = self.x0[:len(blocks)]
        rt.launch(bt, [self.latents[b] for b in blocks], [self.cond_dev] * len(blocks),
                  self.arena, x0s, self.ws)
        for e, x0, (kind, next_pass, next_level) in zip(plan.entries, x0s, posts):
            b = e.block_index
            self.tags[b] = (e.noise_level, self.cond.id)
            if kind == POST_RENOISE:
                eps = self._upload_noise(b, next_pass)
                N.check(N.lib().bc_renoise_f64(N.ptr(x0), N.ptr(eps), next_level,
                                               N.ptr(self.latents[b]), x0.numel(), None,
                                               N.stream_ptr()), "bc_renoise_f64")
            elif kind == POST_EMIT:
                self.final[b] = x0.clone()
                self.latents[b] = self.final[b]
            elif kind == POST_CACHE:
                self.latents.pop(b, None)
            else:  # pragma: no cover
                raise ContractViolation(f"unknown post op {kind}")
        self._mark()

    def recache_block(self, block, mask, vis_list):
        """One causal level-0 forward of an emitted block from its x0 under
        the current conditioning; rewrites its KV slot (recache baseline,
        reference kvpool.py:109-140)."""
        vis = [self.slots.slot_of(v) for v in vis_list]
        slot = self.slots.slot_of(block)
        bt = N.make_batch(self.S, [block], [0.0], [slot], [vis])
        self.rt.launch(bt, [self.final[block]], [self.cond_dev], self.arena, self.x0[:1], self.ws)
        self.tags[block] = (0.0, self.cond.id)

    def begin_stall(self):
        self._stall0 = self.torch.cuda.Event(enable_timing=True)
        self._stall0.record()

    def end_stall(self, iteration):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        self.stalls[iteration] = (self._stall0, ev)

    def kv_handle(self, block):
        level, cid = self.tags[block]
        return SlotKV(self.arena, self.slots.slot_of(block), block, level, cid, self.S)

    def release(self, block):
        self.slots.release(block)

    def emitted_host(self, block):
        self.torch.cuda.current_stream().synchronize()
        self.rt.check_status()
        return self.final[block].cpu().numpy()

    def fill_wall_times(self, events):
        if not events:
            return
        self.torch.cuda.current_stream().synchronize()
        self.rt.check_status()
        first = self.events[0]
        for ev in events:
            i = ev.iteration
            t0, t1 = self.events[i], self.events[i + 1]
            ev.wall_seconds = t0.elapsed_time(t1) / 1e3
            ev.wall_clock = first.elapsed_time(t1) / 1e3
            if i in self.stalls:  # the stall counts on the clock, not in the iteration
                s0, s1 = self.stalls[i]
                ev.wall_seconds -= s0.elapsed_time(s1) / 1e3

    def close(self):
        self.torch.cuda.current_stream().synchronize()
        self._staged.clear()
