"""Multi-GPU temporal parallelism: one process per GPU.

Units are the in-flight blocks of an iteration; a block is owned by rank
``block % world`` for its whole life (so its latents never move -- outputs do
not depend on the placement, the trace keeps the reference's positional
``worker`` label).  Every rank runs the same host loop (scheduler, pool
index, slot allocator are deterministic, so all ranks agree on slots) and
executes only its own entries.  There is one exchange per layer: the q/k
kernel of the owner writes the block's fresh K/V into its slot on *every*
rank (NVLink P2P stores into IPC-mapped peer arenas) and publishes a
``(layer, slot) -> epoch`` flag; a consumer's attention waits for the flag of
a visible slot only before that slot's first key tile.  Pool slots come first
in the ascending gather order, so the transfer overlaps the pool part of the
attention and the summation order is the same for any world size.

Host-side logic here is pure (``owner``, ``rank_entries``, ``need_table``) and
covered by multi-process ``gloo`` tests on CPU; the device part is exercised
on one GPU by :class:`EmulatedRanks`, which steps G rank contexts
layer-interleaved on a single stream.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native as N
from .errors import ContractViolation, InvalidInputError

# Tests flip this to run `workers > 1` sessions as emulated ranks on one GPU.
EMULATE = os.environ.get("BC_EMULATE_RANKS", "0") == "1"


def owner(block: int, world: int) -> int:
    return block % world


def rank_entries(blocks, world: int, rank: int) -> list:
    """Positions (in plan order) of the entries this rank executes."""
    return [i for i, b in enumerate(blocks) if owner(b, world) == rank]


def need_table(local_blocks, vis_lists_local, batch_blocks, slot_epoch: dict, epoch: int,
               world: int, rank: int, slot_of) -> list:
    """Per local entry, per visible block: the flag epoch to wait for before
    reading that slot (0 = written by this rank, stream-ordered).  Fresh
    batch blocks of other ranks need this iteration's epoch; pool blocks
    need the epoch of the iteration that last wrote them (their cache pass)."""
    fresh = set(batch_blocks)
    table = []
    for lst in vis_lists_local:
        row = []
        for vb in lst:
            if owner(vb, world) == rank:
                row.append(0)
            elif vb in fresh:
                row.append(epoch)
            else:
                row.append(int(slot_epoch[slot_of(vb)]))
        table.append(row)
    return table


class SlotEpochs:
    """Epoch of the last write of every arena slot (identical on all ranks)."""

    def __init__(self, n_slots):
        self.epoch = np.zeros(n_slots, dtype=np.int64)

    def __getitem__(self, slot):
        return self.epoch[slot]

    def wrote(self, slots, epoch):
        for s in slots:
            self.epoch[s] = epoch


def make_dist(epoch: int, need_rows, stage: int = -1, layer: int = 0):
    d = N.WanDist()
    d.epoch = epoch
    d.stage = stage
    d.layer = layer
    for e, row in enumerate(need_rows):
        for v, x in enumerate(row):
            d.need[e][v] = int(x)
    return d


class _RankState:
    """Device buffers of one rank: arena, flags, done, counters + context."""

    def __init__(self, weights, cfg, max_entries, n_slots, world, rank, ipc: bool):
        torch = N.torch_mod()
        from .wan import _Ctx
        self.world, self.rank = world, rank
        self.ipc = ipc
        L = cfg.layers
        flag_words = L * n_slots + world + 4
        if ipc:
            self.arena_bytes = L * n_slots * 2 * cfg.tokens_per_block * cfg.model_dim * 2
            self.arena_ptr, self.arena_handle = _ipc_alloc(self.arena_bytes)
            self.flags_ptr, self.flags_handle = _ipc_alloc(flag_words * 4)
            arena = _raw_tensor(self.arena_ptr, (L, n_slots, 2, cfg.tokens_per_block, cfg.model_dim),
                                torch.bfloat16)
        else:
            arena = torch.zeros((L, n_slots, 2, cfg.tokens_per_block, cfg.model_dim),
                                dtype=torch.bfloat16, device="cuda")
            self.flag_buf = torch.zeros(flag_words, dtype=torch.int32, device="cuda")
            self.arena_ptr, self.flags_ptr = N.ptr(arena), N.ptr(self.flag_buf)
        self.ctx = _Ctx(weights, max_entries, n_slots, arena=arena)
        self.L, self.n_slots = L, n_slots

    def my_flags(self):
        return self.flags_ptr

    def my_done(self):
        return self.flags_ptr + 4 * self.L * self.n_slots

    def counters(self):
        return self.my_done() + 4 * self.world

    def attach(self, peers):
        """peers: list of (rank, arena_ptr, flags_ptr) for every other rank."""
        P = N.WanPeers()
        P.n_peers = len(peers)
        P.my_rank = self.rank
        P.n_ranks = self.world
        for i, (r, arena, flags) in enumerate(peers):
            P.peer_arena[i] = arena
            P.peer_flags[i] = flags
            P.peer_done[i] = flags + 4 * self.L * self.n_slots
        P.my_flags = self.my_flags()
        P.my_done = self.my_done()
        P.counters = self.counters()
        N.check(N.lib().bc_wan_set_peers(self.ctx.handle, P), "bc_wan_set_peers")


def _ipc_alloc(nbytes):
    ptr = ctypes.c_void_p()
    handle = ctypes.create_string_buffer(64)
    N.check(N.lib().bc_ipc_malloc(int(nbytes), ctypes.byref(ptr), handle), "bc_ipc_malloc")
    return ptr.value, handle.raw


def _ipc_open(handle: bytes):
    ptr = ctypes.c_void_p()
    N.check(N.lib().bc_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(ptr)), "bc_ipc_open")
    return ptr.value


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def _raw_tensor(ptr, shape, dtype):
    torch = N.torch_mod()
    typestr = {torch.bfloat16: "<f2", torch.float32: "<f4", torch.int32: "<i4"}[dtype]
    t = torch.as_tensor(_CudaArray(ptr, shape, typestr), device="cuda")
    return t.view(dtype) if dtype == torch.bfloat16 else t


class DistWanSession:
    """Engine session for one rank of a torch.distributed job (one GPU per
    process).  Implements the same protocol as :class:`wan.WanSession`."""

    def __init__(self, rt, config, conditioning, session_seed, noise_feed=None):
        import torch.distributed as dist
        from .kvpool import SlotAllocator
        from .wan import HostNoiseFeed
        torch = N.torch_mod()
        self.torch, self.dist = torch, dist
        self.cfg = config
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        width = min(config.cascade_width, config.num_blocks)
        n_slots = config.window_blocks + config.sink_blocks + width + 1
        self.state = _RankState(rt.weights, config, width, n_slots, self.world, self.rank, ipc=True)
        mine = (self.rank, self.state.arena_handle, self.state.flags_handle)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine)
        self._opened = []
        peers = []
        for r, ah, fh in everyone:
            if r == self.rank:
                continue
            a, f = _ipc_open(ah), _ipc_open(fh)
            self._opened += [a, f]
            peers.append((r, a, f))
        self.state.attach(peers)
        dist.barrier()
        self.slots = SlotAllocator(n_slots)
        self.slot_epoch = SlotEpochs(n_slots)
        self.shape = (config.block_size, config.latent_channels, config.latent_height,
                      config.latent_width)
        self.noise = noise_feed if noise_feed is not None else HostNoiseFeed(session_seed, config)
        self.latents, self.final, self.tags, self.host_out = {}, {}, {}, {}
        # one pinned staging area for every emitted block (no per-emission
        # cudaHostAlloc, which would serialise against the device)
        self.host_buf = torch.empty((config.num_blocks,) + tuple(self.shape),
                                    dtype=torch.float32).pin_memory()
        self.eps = [torch.empty(self.shape, dtype=torch.float32, device="cuda") for _ in range(width)]
        self.events = []
        self.set_conditioning(conditioning)
        self._mark()

    def _mark(self):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append(ev)

    def recache_block(self, block, mask, vis_list):
        raise InvalidInputError("the KV-recache comparison baseline runs on one GPU only "
                                "(the product switch is mode='cascade')")

    def begin_stall(self):
        pass

    def end_stall(self, iteration):
        pass

    def set_conditioning(self, cond):
        self.cond = cond
        self.state.ctx.set_text(cond)

    def step(self, plan, mask, pool, vis_lists, posts):
        from .wan import POST_CACHE, POST_EMIT, POST_RENOISE, _make_update
        torch = self.torch
        epoch = plan.iteration + 1
        blocks = plan.blocks
        for b in blocks:
            self.slots.acquire(b)
        local = rank_entries(blocks, self.world, self.rank)
        if not local:
            N.check(N.lib().bc_wan_signal_done(self.state.ctx.handle, epoch, N.stream_ptr()),
                    "bc_wan_signal_done")
        else:
            init_req, init_dst, eps_req, eps_dst, eps_ptrs, outs, nexts = [], [], [], [], [], [], []
            for k, i in enumerate(local):
                e = plan.entries[i]
                kind, next_pass, next_level = posts[i]
                if e.pass_index == 0 and e.block_index not in self.latents:
                    t = torch.empty(self.shape, dtype=torch.float32, device="cuda")
                    self.latents[e.block_index] = t
                    init_req.append((e.block_index, 0))
                    init_dst.append(t)
                if kind == POST_RENOISE:
                    eps_req.append((e.block_index, next_pass))
                    eps_dst.append(self.eps[k])
                    eps_ptrs.append(self.eps[k])
                else:
                    eps_ptrs.append(None)
                if kind == POST_EMIT:
                    out = torch.empty(self.shape, dtype=torch.float32, device="cuda")
                    self.final[e.block_index] = out
                    outs.append(out)
                else:
                    outs.append(None)
                nexts.append(next_level)
            if init_req or eps_req:
                self.noise.fetch(init_req + eps_req, init_dst + eps_dst)
            lb = [blocks[i] for i in local]
            vis_local = [vis_lists[i] for i in local]
            bt = N.make_batch(self.cfg.block_size, lb, [plan.entries[i].noise_level for i in local],
                              [self.slots.slot_of(b) for b in lb],
                              [[self.slots.slot_of(v) for v in lst] for lst in vis_local])
            need = need_table(lb, vis_local, blocks, self.slot_epoch, epoch, self.world, self.rank,
                              self.slots.slot_of)
            upd = _make_update([posts[i][0] for i in local], [self.latents[b] for b in lb], eps_ptrs,
                               outs, nexts)
            N.check(N.lib().bc_wan_step_dist(self.state.ctx.handle, bt, upd, make_dist(epoch, need),
                                             N.ptr(self.state.ctx.status), N.stream_ptr()),
                    "bc_wan_step_dist")
            for k, i in enumerate(local):
                e = plan.entries[i]
                if posts[i][0] == POST_EMIT:
                    host = self.host_buf[e.block_index]
                    host.copy_(self.final[e.block_index], non_blocking=True)
                    self.host_out[e.block_index] = host
                elif posts[i][0] == POST_CACHE:
                    self.latents.pop(e.block_index, None)
        self.slot_epoch.wrote([self.slots.slot_of(b) for b in blocks], epoch)
        for e in plan.entries:
            self.tags[e.block_index] = (e.noise_level, self.cond.id)
        self._mark()

    def kv_handle(self, block):
        from .kvpool import SlotKV
        level, cid = self.tags[block]
        return SlotKV(self.state.ctx, self.slots.slot_of(block), block, level, cid, self.cfg.block_size)

    def release(self, block):
        self.slots.release(block)

    def emitted_host(self, block):
        self.torch.cuda.current_stream().synchronize()
        self.state.ctx.check_status()
        if block in self.host_out:
            return self.host_out[block].numpy().reshape(self.cfg.block_size, -1).astype(np.float64)
        return None

    def gather_outputs(self, blocks):
        """Every rank gets every emitted block (owner -> all)."""
        mine = {b: self.emitted_host(b) for b in blocks if owner(b, self.world) == self.rank}
        parts = [None] * self.world
        self.dist.all_gather_object(parts, mine)
        out = {}
        for p in parts:
            out.update(p)
        return out

    def fill_wall_times(self, events):
        if not events:
            return
        self.torch.cuda.current_stream().synchronize()
        self.state.ctx.check_status()
        first = self.events[0]
        for ev in events:
            t0, t1 = self.events[ev.iteration], self.events[ev.iteration + 1]
            ev.wall_seconds = t0.elapsed_time(t1) / 1e3
            ev.wall_clock = first.elapsed_time(t1) / 1e3

    def close(self):
        self.torch.cuda.synchronize()
        self.dist.barrier()
        for p in self._opened:
            N.lib().bc_ipc_close(p)
        self._opened = []
        self.state.ctx.close()
        N.lib().bc_free(self.state.arena_ptr)
        N.lib().bc_free(self.state.flags_ptr)


class EmulatedRanks:
    """G rank contexts on ONE GPU, stepped layer-interleaved on one stream:
    every rank's stage 0, then for each layer all ranks' part A (K/V write +
    peer push + flag publish) before any rank's part B (attention waits on
    the flags), then all ranks' stage 3.  Exercises exactly the device code
    of the multi-GPU path (P2P pushes become same-device stores)."""

    def __init__(self, rt, config, conditioning, session_seed, world, noise_feed=None):
        from .kvpool import SlotAllocator
        from .wan import HostNoiseFeed
        torch = N.torch_mod()
        self.torch, self.cfg, self.world = torch, config, world
        width = min(config.cascade_width, config.num_blocks)
        n_slots = config.window_blocks + config.sink_blocks + width + 1
        self.ranks = [_RankState(rt.weights, config, width, n_slots, world, r, ipc=False)
                      for r in range(world)]
        for st in self.ranks:
            st.attach([(o.rank, o.arena_ptr, o.flags_ptr) for o in self.ranks if o.rank != st.rank])
        self.slots = SlotAllocator(n_slots)
        self.slot_epoch = SlotEpochs(n_slots)
        self.shape = (config.block_size, config.latent_channels, config.latent_height,
                      config.latent_width)
        self.noise = noise_feed if noise_feed is not None else HostNoiseFeed(session_seed, config)
        self.latents, self.final, self.tags, self.host_out = {}, {}, {}, {}
        # one pinned staging area for every emitted block (no per-emission
        # cudaHostAlloc, which would serialise against the device)
        self.host_buf = torch.empty((config.num_blocks,) + tuple(self.shape),
                                    dtype=torch.float32).pin_memory()
        self.eps = [torch.empty(self.shape, dtype=torch.float32, device="cuda")
                    for _ in range(width * world)]
        self.events = []
        self.set_conditioning(conditioning)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append(ev)

    def recache_block(self, block, mask, vis_list):
        raise InvalidInputError("the KV-recache comparison baseline runs on one GPU only "
                                "(the product switch is mode='cascade')")

    def begin_stall(self):
        pass

    def end_stall(self, iteration):
        pass

    def set_conditioning(self, cond):
        self.cond = cond
        for st in self.ranks:
            st.ctx.set_text(cond)

    def step(self, plan, mask, pool, vis_lists, posts):
        from .wan import POST_CACHE, POST_EMIT, POST_RENOISE, _make_update
        torch = self.torch
        epoch = plan.iteration + 1
        blocks = plan.blocks
        for b in blocks:
            self.slots.acquire(b)
        work = []
        init_req, init_dst, eps_req, eps_dst = [], [], [], []
        for r, st in enumerate(self.ranks):
            local = rank_entries(blocks, self.world, r)
            if not local:
                work.append((st, None))
                continue
            eps_ptrs, outs, nexts = [], [], []
            for k, i in enumerate(local):
                e = plan.entries[i]
                kind, next_pass, next_level = posts[i]
                if e.pass_index == 0 and e.block_index not in self.latents:
                    t = torch.empty(self.shape, dtype=torch.float32, device="cuda")
                    self.latents[e.block_index] = t
                    init_req.append((e.block_index, 0))
                    init_dst.append(t)
                if kind == POST_RENOISE:
                    buf = self.eps[r * len(self.eps) // self.world + k]
                    eps_req.append((e.block_index, next_pass))
                    eps_dst.append(buf)
                    eps_ptrs.append(buf)
                else:
                    eps_ptrs.append(None)
                if kind == POST_EMIT:
                    out = torch.empty(self.shape, dtype=torch.float32, device="cuda")
                    self.final[e.block_index] = out
                    outs.append(out)
                else:
                    outs.append(None)
                nexts.append(next_level)
            lb = [blocks[i] for i in local]
            vis_local = [vis_lists[i] for i in local]
            bt = N.make_batch(self.cfg.block_size, lb, [plan.entries[i].noise_level for i in local],
                              [self.slots.slot_of(b) for b in lb],
                              [[self.slots.slot_of(v) for v in lst] for lst in vis_local])
            need = need_table(lb, vis_local, blocks, self.slot_epoch, epoch, self.world, r,
                              self.slots.slot_of)
            upd = _make_update([posts[i][0] for i in local], [self.latents[b] for b in lb], eps_ptrs,
                               outs, nexts)
            work.append((st, (bt, upd, need)))
        if init_req or eps_req:
            self.noise.fetch(init_req + eps_req, init_dst + eps_dst)
        sp = N.stream_ptr()
        lib = N.lib()

        def run(st, item, stage, layer=0):
            bt, upd, need = item
            N.check(lib.bc_wan_step_dist(st.ctx.handle, bt, upd, make_dist(epoch, need, stage, layer),
                                         N.ptr(st.ctx.status), sp), "bc_wan_step_dist")

        for st, item in work:
            if item is not None:
                run(st, item, 0)
        for layer in range(self.cfg.layers):
            for st, item in work:
                if item is not None:
                    run(st, item, 1, layer)
            for st, item in work:
                if item is not None:
                    run(st, item, 2, layer)
        for st, item in work:
            if item is not None:
                run(st, item, 3)
            else:
                N.check(lib.bc_wan_signal_done(st.ctx.handle, epoch, sp), "bc_wan_signal_done")
        for e, (kind, _, _) in zip(plan.entries, posts):
            self.tags[e.block_index] = (e.noise_level, self.cond.id)
            if kind == POST_EMIT:
                host = self.host_buf[e.block_index]
                host.copy_(self.final[e.block_index], non_blocking=True)
                self.host_out[e.block_index] = host
            elif kind == POST_CACHE:
                self.latents.pop(e.block_index, None)
        self.slot_epoch.wrote([self.slots.slot_of(b) for b in blocks], epoch)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append(ev)

    def kv_handle(self, block):
        from .kvpool import SlotKV
        level, cid = self.tags[block]
        return SlotKV(self.ranks[0].ctx, self.slots.slot_of(block), block, level, cid,
                      self.cfg.block_size)

    def release(self, block):
        self.slots.release(block)

    def emitted_host(self, block):
        self.torch.cuda.current_stream().synchronize()
        for st in self.ranks:
            st.ctx.check_status()
        return self.host_out[block].numpy().reshape(self.cfg.block_size, -1).astype(np.float64)

    def fill_wall_times(self, events):
        if not events:
            return
        self.torch.cuda.current_stream().synchronize()
        first = self.events[0]
        for ev in events:
            t0, t1 = self.events[ev.iteration], self.events[ev.iteration + 1]
            ev.wall_seconds = t0.elapsed_time(t1) / 1e3
            ev.wall_clock = first.elapsed_time(t1) / 1e3

    def replica_arenas(self):
        return [st.ctx.arena for st in self.ranks]

    def close(self):
        for st in self.ranks:
            st.ctx.close()
