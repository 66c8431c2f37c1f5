"""Multi-GPU temporal parallelism: one process
per GPU.

Every rank runs the same host loop (scheduler, pool index and slot
allocator are deterministic, so all ranks agree on slots) and keeps a full
KV-arena replica.  An iteration's work is partitioned in one of two ways
(``BC_TEMPORAL_SHARD``):

* ``rows`` (default): every rank runs EVERY in-flight entry, but only a
  contiguous slice of the batch's n*T concatenated query rows (balanced in
  128-row query tiles, :func:`row_slices`).  Any world size is load
  balanced, including G > cascade width (8 GPUs for a width-5 cascade) and
  the fill/drain iterations.  A rank's fresh K/V rows go to every peer
  replica; its head-GEMM rows (Y, 64 floats per token) go to every peer's
  Y; every rank then applies the same flow->x0 + renoise to every entry, so
  latents are replicated and never move.
* ``blocks``: block ``b`` is executed by rank ``b % world`` for its whole
  life (whole entries per rank; ranks beyond the width idle).

In both, the exchange is one per layer: fresh K/V rows reach the peers'
replicas over NVLink (P2P stores from the q/k kernel, whose last CTA
publishes ``flags[layer][slot][producer] = epoch``), and a consumer's attention waits
for the flags of a visible slot's producers only before that slot's first
key tile.  Pool slots come first in the ascending gather order, so the
transfer overlaps the pool part of the attention, and the summation order
(and every row's arithmetic) is the same for any world size: outputs are
bit-identical for every G and either partition.

Host-side logic here is pure (``owner``, ``rank_entries``, ``row_slices``,
``need_table``) and covered by multi-process ``gloo`` tests on CPU; the
device part is exercised on one GPU by :class:`EmulatedRanks`, which steps G
rank contexts stage-interleaved on a single stream.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native as N
from .errors import ContractViolation, InvalidInputError

# Tests flip this to run `workers > 1` sessions as emulated ranks on one GPU.
EMULATE = os.environ.get("BC_EMULATE_RANKS", "0") == "1"
# Process group of the denoiser ranks when the job also has a decode rank
# (decode_rank.split_ranks); None: the whole world group denoises.
DIT_GROUP = None


def dit_world() -> int:
    """Denoiser ranks of the initialised torch.distributed job (0: none)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 0
    return dist.get_world_size(DIT_GROUP)
ROW_TILE = 128  # query rows per attention tile: the unit of the rows partition
ROW_UNIT_SMALL = 16  # unit when a batch has fewer than 2 tiles per rank


def shard_mode() -> str:
    m = os.environ.get("BC_TEMPORAL_SHARD", "rows")
    if m not in ("rows", "blocks"):
        raise InvalidInputError(f"BC_TEMPORAL_SHARD must be 'rows' or 'blocks', not {m!r}")
    return m


def owner(block: int, world: int) -> int:
    return block % world


def rank_entries(blocks, world: int, rank: int) -> list:
    """blocks partition: positions (in plan order) of this rank's entries."""
    return [i for i, b in enumerate(blocks) if owner(b, world) == rank]


def row_slices(n: int, T: int, world: int) -> list:
    """rows partition: per rank the global row slice [r0, r1) of the n*T
    concatenated rows.  The unit is a query tile (128 rows, the last tile of
    an entry shorter); rank r gets tiles [r*K/G, (r+1)*K/G).  Tiny blocks
    (fewer than 2 tiles per rank) fall back to 16-row units so every rank
    still gets rows.  An empty slice is (n*T, n*T)."""
    unit = ROW_TILE if n * -(-T // ROW_TILE) >= 2 * world else ROW_UNIT_SMALL
    tiles = [(e * T + t, e * T + min(t + unit, T)) for e in range(n) for t in range(0, T, unit)]
    K = len(tiles)
    out = []
    for r in range(world):
        a, b = r * K // world, (r + 1) * K // world
        out.append((tiles[a][0], tiles[b - 1][1]) if b > a else (n * T, n * T))
    return out


def entry_producers(slices, n: int, T: int) -> list:
    """rows partition: per entry position, the bit mask of ranks whose slice
    holds some of its rows (they write its K/V)."""
    masks = []
    for i in range(n):
        lo, hi = i * T, (i + 1) * T
        m = 0
        for r, (a, b) in enumerate(slices):
            if a < hi and b > lo:
                m |= 1 << r
        masks.append(m)
    return masks


class SlotEpochs:
    """Epoch of the last write of every arena slot and the ranks that wrote
    it (identical on all ranks)."""

    def __init__(self, n_slots):
        self.epoch = np.zeros(n_slots, dtype=np.int64)
        self.mask = np.zeros(n_slots, dtype=np.int64)

    def __getitem__(self, slot):
        return self.epoch[slot]

    def wrote(self, slots, epoch, masks=None):
        for i, s in enumerate(slots):
            self.epoch[s] = epoch
            if masks is not None:
                self.mask[s] = masks[i]


def need_table(local_blocks, vis_lists_local, batch_blocks, slot_epoch: SlotEpochs, epoch: int,
               world: int, rank: int, slot_of, producers=None) -> tuple:
    """Per local entry, per visible block: (epoch to wait for, producer-rank
    mask) before reading that slot.  Rows written by this rank are stream-
    ordered (not in the mask).  Fresh batch blocks need this iteration's
    epoch from their producers this iteration; pool blocks need the epoch of
    the iteration that last wrote them, from the ranks that wrote it then.
    ``producers``: block -> mask this iteration (rows partition); None =
    blocks partition (the owner is the only producer)."""
    fresh = set(batch_blocks)
    me = 1 << rank
    need, pmask = [], []
    for lst in vis_lists_local:
        nrow, mrow = [], []
        for vb in lst:
            s = slot_of(vb)
            if producers is None:
                m = (1 << owner(vb, world)) & ~me
                ep = epoch if vb in fresh else int(slot_epoch[s])
            elif vb in fresh:
                m, ep = producers[vb] & ~me, epoch
            else:
                m, ep = int(slot_epoch.mask[s]) & ~me, int(slot_epoch[s])
            nrow.append(ep if m else 0)
            mrow.append(m if m else 0)
        need.append(nrow)
        pmask.append(mrow)
    return need, pmask


def make_dist(epoch: int, need_rows, pmask_rows, stage: int = -1, layer: int = 0, rows=None):
    d = N.WanDist()
    d.epoch = epoch
    d.stage = stage
    d.layer = layer
    for e, (nrow, mrow) in enumerate(zip(need_rows, pmask_rows)):
        for v, (x, m) in enumerate(zip(nrow, mrow)):
            d.need[e][v] = int(x)
            d.pmask[e][v] = int(m)
    if rows is not None:
        d.row0, d.row1 = rows
    return d


def flag_layout(L: int, n_slots: int, world: int) -> dict:
    """u32 word offsets in a rank's flag buffer:
    [L][n_slots][world] K/V ready | done[world] | yready[world] | counters[4]."""
    kv = L * n_slots * world
    return {"done": kv, "yready": kv + world, "counters": kv + 2 * world, "words": kv + 2 * world + 4}


class _RankState:
    """Device buffers of one rank: arena, flags (+done, yready, counters), Y
    (rows partition) + context."""

    def __init__(self, weights, cfg, max_entries, n_slots, world, rank, ipc: bool):
        torch = N.torch_mod()
        from .wan import _Ctx
        self.world, self.rank = world, rank
        self.ipc = ipc
        L = cfg.layers
        self.lay = flag_layout(L, n_slots, world)
        y_bytes = max_entries * cfg.tokens_per_block * 64 * 4
        if ipc:
            self.arena_bytes = L * n_slots * 2 * cfg.tokens_per_block * cfg.model_dim * 2
            self.arena_ptr, self.arena_handle = _ipc_alloc(self.arena_bytes)
            self.flags_ptr, self.flags_handle = _ipc_alloc(self.lay["words"] * 4)
            self.y_ptr, self.y_handle = _ipc_alloc(y_bytes)
            arena = _raw_tensor(self.arena_ptr, (L, n_slots, 2, cfg.tokens_per_block, cfg.model_dim),
                                torch.bfloat16)
        else:
            arena = torch.zeros((L, n_slots, 2, cfg.tokens_per_block, cfg.model_dim),
                                dtype=torch.bfloat16, device="cuda")
            self.flag_buf = torch.zeros(self.lay["words"], dtype=torch.int32, device="cuda")
            self.y_buf = torch.zeros(y_bytes // 4, dtype=torch.float32, device="cuda")
            self.arena_ptr, self.flags_ptr = N.ptr(arena), N.ptr(self.flag_buf)
            self.y_ptr = N.ptr(self.y_buf)
        self.ctx = _Ctx(weights, max_entries, n_slots, arena=arena)
        self.L, self.n_slots = L, n_slots

    def word(self, name, base=None):
        return (self.flags_ptr if base is None else base) + 4 * self.lay[name]

    def attach(self, peers, rows: bool):
        """peers: list of (rank, arena_ptr, flags_ptr, y_ptr) for every other rank."""
        P = N.WanPeers()
        P.n_peers = len(peers)
        P.my_rank = self.rank
        P.n_ranks = self.world
        for i, (r, arena, flags, y) in enumerate(peers):
            P.peer_arena[i] = arena
            P.peer_flags[i] = flags
            P.peer_done[i] = self.word("done", flags)
            if rows:
                P.peer_y[i] = y
                P.peer_yready[i] = self.word("yready", flags)
        P.my_flags = self.flags_ptr
        P.my_done = self.word("done")
        P.counters = self.word("counters")
        if rows:
            P.my_y = self.y_ptr
            P.my_yready = self.word("yready")
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


class _RankWork:
    """Host-side step description of one rank (shared by the real and the
    emulated multi-rank sessions)."""

    def __init__(self, mode, plan, vis_lists, world, rank, slots, slot_epoch, epoch, T):
        blocks = plan.blocks
        n = len(blocks)
        self.rows = None
        producers = None
        if mode == "rows":
            sl = row_slices(n, T, world)
            masks = entry_producers(sl, n, T)
            producers = dict(zip(blocks, masks))
            self.local = list(range(n))
            self.rows = sl[rank]
            self.masks = masks
        else:
            self.local = rank_entries(blocks, world, rank)
            self.masks = [1 << owner(b, world) for b in blocks]
        lb = [blocks[i] for i in self.local]
        vis_local = [vis_lists[i] for i in self.local]
        self.blocks = lb
        self.need, self.pmask = need_table(lb, vis_local, blocks, slot_epoch, epoch, world, rank,
                                           slots.slot_of, producers)
        self.vis_local = vis_local
        self.epoch = epoch

    def dist(self, stage=-1, layer=0):
        return make_dist(self.epoch, self.need, self.pmask, stage, layer, self.rows)


class _Replica:
    """Per-rank latents / noise / outputs of a session.  In the rows
    partition every rank holds every in-flight block's latents (it applies
    the same update to all of them); in the blocks partition only its own."""

    def __init__(self, torch, cfg, width):
        self.torch = torch
        self.shape = (cfg.block_size, cfg.latent_channels, cfg.latent_height, cfg.latent_width)
        self.latents, self.final = {}, {}
        self.eps = [torch.empty(self.shape, dtype=torch.float32, device="cuda") for _ in range(width)]

    def prepare(self, plan, posts, local, init_req, init_dst, eps_req, eps_dst):
        """Allocates this step's buffers; returns (latents, eps, outs, next_levels) per local entry."""
        from .wan import POST_EMIT, POST_RENOISE
        torch = self.torch
        lats, eps, outs, nexts = [], [], [], []
        for k, i in enumerate(local):
            e = plan.entries[i]
            kind, next_pass, next_level = posts[i]
            b = e.block_index
            if e.pass_index == 0 and b not in self.latents:
                t = torch.empty(self.shape, dtype=torch.float32, device="cuda")
                self.latents[b] = t
                init_req.append((b, 0))
                init_dst.append(t)
            lats.append(self.latents[b])
            if kind == POST_RENOISE:
                eps_req.append((b, next_pass))
                eps_dst.append(self.eps[k])
                eps.append(self.eps[k])
            else:
                eps.append(None)
            if kind == POST_EMIT:
                out = torch.empty(self.shape, dtype=torch.float32, device="cuda")
                self.final[b] = out
                outs.append(out)
            else:
                outs.append(None)
            nexts.append(next_level)
        return lats, eps, outs, nexts

    def retire(self, plan, posts, local):
        from .wan import POST_CACHE
        for i in local:
            if posts[i][0] == POST_CACHE:
                self.latents.pop(plan.entries[i].block_index, None)


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
        self.mode = shard_mode()
        self.group = DIT_GROUP
        self.world, self.rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        width = min(config.cascade_width, config.num_blocks)
        n_slots = config.window_blocks + config.sink_blocks + width + 1
        self.state = _RankState(rt.weights, config, width, n_slots, self.world, self.rank, ipc=True)
        mine = (self.rank, self.state.arena_handle, self.state.flags_handle, self.state.y_handle)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=self.group)
        self._opened = []
        peers = []
        for r, ah, fh, yh in everyone:
            if r == self.rank:
                continue
            a, f, y = _ipc_open(ah), _ipc_open(fh), _ipc_open(yh)
            self._opened += [a, f, y]
            peers.append((r, a, f, y))
        self.state.attach(peers, rows=self.mode == "rows")
        dist.barrier(group=self.group)
        self.slots = SlotAllocator(n_slots)
        self.slot_epoch = SlotEpochs(n_slots)
        self.rep = _Replica(torch, config, width)
        self.shape = self.rep.shape
        self.noise = noise_feed if noise_feed is not None else HostNoiseFeed(session_seed, config)
        self.tags, self.host_out = {}, {}
        self.host_pending, self.host_f64 = {}, {}
        # one pinned staging area for every emitted block (no per-emission
        # cudaHostAlloc, which would serialise against the device)
        self.host_buf = torch.empty((config.num_blocks,) + tuple(self.shape),
                                    dtype=torch.float32, pin_memory=True)
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
        from .wan import POST_EMIT, _make_update
        self._convert_landed()
        epoch = plan.iteration + 1
        blocks = plan.blocks
        for b in blocks:
            self.slots.acquire(b)
        work = _RankWork(self.mode, plan, vis_lists, self.world, self.rank, self.slots,
                         self.slot_epoch, epoch, self.cfg.tokens_per_block)
        if not work.local:
            N.check(N.lib().bc_wan_signal_done(self.state.ctx.handle, epoch, N.stream_ptr()),
                    "bc_wan_signal_done")
        else:
            init_req, init_dst, eps_req, eps_dst = [], [], [], []
            lats, eps, outs, nexts = self.rep.prepare(plan, posts, work.local, init_req, init_dst,
                                                      eps_req, eps_dst)
            if init_req or eps_req:
                self._fetch_noise(init_req + eps_req, init_dst + eps_dst)
            bt = N.make_batch(self.cfg.block_size, work.blocks,
                              [plan.entries[i].noise_level for i in work.local],
                              [self.slots.slot_of(b) for b in work.blocks],
                              [[self.slots.slot_of(v) for v in lst] for lst in work.vis_local])
            upd = _make_update([posts[i][0] for i in work.local], lats, eps, outs, nexts)
            N.check(N.lib().bc_wan_step_dist(self.state.ctx.handle, bt, upd, work.dist(),
                                             N.ptr(self.state.ctx.status), N.stream_ptr()),
                    "bc_wan_step_dist")
            for i in work.local:
                b = plan.entries[i].block_index
                if posts[i][0] == POST_EMIT:
                    host = self.host_buf[b]
                    host.copy_(self.rep.final[b], non_blocking=True)
                    self.host_out[b] = host
                    self.host_f64.pop(b, None)
                    ev = self.torch.cuda.Event()
                    ev.record()
                    self.host_pending[b] = ev
            self.rep.retire(plan, posts, work.local)
        self.slot_epoch.wrote([self.slots.slot_of(b) for b in blocks], epoch, work.masks)
        for e in plan.entries:
            self.tags[e.block_index] = (e.noise_level, self.cond.id)
        self._mark()

    def _fetch_noise(self, keys, dests):
        """Counter-keyed noise for this step.  In the rows partition every
        rank needs every entry's noise; with NCCL the host generation is
        split round-robin over the ranks and the draws are all-gathered on
        the device (a few MB per iteration) instead of every rank drawing
        all of them on the node's shared host cores.  Bit-identical either
        way: each key's draw is a pure function of the key."""
        dist, torch = self.dist, self.torch
        nccl = dist.get_backend(self.group) == "nccl"
        forced = os.environ.get("BC_NOISE_GATHER") == "1"   # test hook (gloo: gathers on the host)
        if self.mode != "rows" or not (nccl or forced) or not hasattr(self.noise, "stream"):
            self.noise.fetch(keys, dests)
            return
        G = self.world
        chunk = -(-len(keys) // G)
        mine = keys[self.rank::G]
        where = "cuda" if nccl else "cpu"
        buf = torch.zeros((chunk,) + tuple(self.shape), dtype=torch.float32, device=where)
        if mine:
            self.noise.fetch(mine, [buf[i] for i in range(len(mine))])
            if where == "cpu":
                torch.cuda.current_stream().synchronize()
        gathered = torch.empty((G * chunk,) + tuple(self.shape), dtype=torch.float32, device=where)
        dist.all_gather_into_tensor(gathered, buf, group=self.group)
        for i, dst in enumerate(dests):   # key i was drawn by rank i % G as its (i // G)-th
            dst.copy_(gathered[(i % G) * chunk + i // G], non_blocking=where == "cuda")

    def kv_handle(self, block):
        from .kvpool import SlotKV
        level, cid = self.tags[block]
        return SlotKV(self.state.ctx, self.slots.slot_of(block), block, level, cid, self.cfg.block_size)

    def release(self, block):
        self.slots.release(block)

    def _convert_landed(self):
        # float64 conversion of emitted blocks whose D2H copy has landed,
        # while the device runs (as WanSession does)
        for b, ev in list(self.host_pending.items()):
            if ev.query():
                self.host_f64[b] = self.host_out[b].numpy().reshape(self.cfg.block_size, -1).astype(np.float64)
                del self.host_pending[b]

    def emitted_host(self, block):
        self.torch.cuda.current_stream().synchronize()
        self.state.ctx.check_status()
        self.host_pending.pop(block, None)
        cached = self.host_f64.pop(block, None)
        if cached is not None:
            return cached
        if block in self.host_out:
            return self.host_out[block].numpy().reshape(self.cfg.block_size, -1).astype(np.float64)
        return None

    def emitted_device(self, block):
        """The emitted block's x0 on this rank's device (every rank has every
        block in the rows partition; in the blocks partition only its owner)."""
        t = self.rep.final.get(block)
        if t is None:
            raise ContractViolation(f"block {block} was not emitted on rank {self.rank} "
                                    f"(blocks partition: rank {owner(block, self.world)} owns it)")
        return t

    def gather_outputs(self, blocks):
        """Every rank gets every emitted block (rows: already replicated;
        blocks: owner -> all)."""
        if self.mode == "rows":
            return {b: self.emitted_host(b) for b in blocks}
        mine = {b: self.emitted_host(b) for b in blocks if owner(b, self.world) == self.rank}
        parts = [None] * self.world
        self.dist.all_gather_object(parts, mine, group=self.group)
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
        self.dist.barrier(group=self.group)
        for p in self._opened:
            N.lib().bc_ipc_close(p)
        self._opened = []
        self.state.ctx.close()
        for p in (self.state.arena_ptr, self.state.flags_ptr, self.state.y_ptr):
            N.lib().bc_free(p)


class EmulatedRanks:
    """G rank contexts on ONE GPU, stepped stage-interleaved on one stream:
    every rank's stage 0, then for each layer all ranks' part A (K/V write +
    peer push + flag publish) before any rank's part B (attention waits on
    the flags), then all ranks' head (+ Y push), then all ranks' update.
    Exercises exactly the device code of the multi-GPU path (P2P pushes
    become same-device copies); each rank has its own latents replica."""

    def __init__(self, rt, config, conditioning, session_seed, world, noise_feed=None):
        from .kvpool import SlotAllocator
        from .wan import HostNoiseFeed
        torch = N.torch_mod()
        self.torch, self.cfg, self.world = torch, config, world
        self.mode = shard_mode()
        width = min(config.cascade_width, config.num_blocks)
        n_slots = config.window_blocks + config.sink_blocks + width + 1
        self.ranks = [_RankState(rt.weights, config, width, n_slots, world, r, ipc=False)
                      for r in range(world)]
        for st in self.ranks:
            st.attach([(o.rank, o.arena_ptr, o.flags_ptr, o.y_ptr) for o in self.ranks if o.rank != st.rank],
                      rows=self.mode == "rows")
        self.slots = SlotAllocator(n_slots)
        self.slot_epoch = SlotEpochs(n_slots)
        self.reps = [_Replica(torch, config, width) for _ in range(world)]
        self.shape = self.reps[0].shape
        # BC_EMULATE_TIMING=1: per iteration, each rank's own device time (ms)
        self.rank_times = [] if os.environ.get("BC_EMULATE_TIMING") == "1" else None
        self.noise = noise_feed if noise_feed is not None else HostNoiseFeed(session_seed, config)
        self.tags, self.host_out = {}, {}
        # one pinned staging area for every emitted block (no per-emission
        # cudaHostAlloc, which would serialise against the device)
        self.host_buf = torch.empty((config.num_blocks,) + tuple(self.shape),
                                    dtype=torch.float32, pin_memory=True)
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
        from .wan import POST_EMIT, _make_update
        torch = self.torch
        epoch = plan.iteration + 1
        blocks = plan.blocks
        for b in blocks:
            self.slots.acquire(b)
        items = []
        init_req, init_dst, eps_req, eps_dst = [], [], [], []
        for r, st in enumerate(self.ranks):
            work = _RankWork(self.mode, plan, vis_lists, self.world, r, self.slots,
                             self.slot_epoch, epoch, self.cfg.tokens_per_block)
            if not work.local:
                items.append((st, work, None, None))
                continue
            lats, eps, outs, nexts = self.reps[r].prepare(plan, posts, work.local, init_req, init_dst,
                                                          eps_req, eps_dst)
            bt = N.make_batch(self.cfg.block_size, work.blocks,
                              [plan.entries[i].noise_level for i in work.local],
                              [self.slots.slot_of(b) for b in work.blocks],
                              [[self.slots.slot_of(v) for v in lst] for lst in work.vis_local])
            upd = _make_update([posts[i][0] for i in work.local], lats, eps, outs, nexts)
            items.append((st, work, bt, upd))
        if init_req or eps_req:
            self.noise.fetch(init_req + eps_req, init_dst + eps_dst)
        sp = N.stream_ptr()
        lib = N.lib()

        timing = self.rank_times is not None
        marks = {}

        def run(st, work, bt, upd, stage, layer=0):
            if timing:  # device time of this rank's own kernels (the work one GPU would do)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            N.check(lib.bc_wan_step_dist(st.ctx.handle, bt, upd, work.dist(stage, layer),
                                         N.ptr(st.ctx.status), sp), "bc_wan_step_dist")
            if timing:
                e1.record()
                marks.setdefault(st.rank, []).append((e0, e1))

        live = [it for it in items if it[2] is not None]
        for it in live:
            run(*it, 0)
        for layer in range(self.cfg.layers):
            for it in live:
                run(*it, 1, layer)
            for it in live:
                run(*it, 2, layer)
        for it in live:
            run(*it, 3)
        for it in live:
            run(*it, 4)
        for st, work, bt, _ in items:
            if bt is None:
                N.check(lib.bc_wan_signal_done(st.ctx.handle, epoch, sp), "bc_wan_signal_done")
        for r, (st, work, bt, _) in enumerate(items):
            if bt is None:
                continue
            for i in work.local:
                b = plan.entries[i].block_index
                if posts[i][0] == POST_EMIT and b not in self.host_out:
                    host = self.host_buf[b]
                    host.copy_(self.reps[r].final[b], non_blocking=True)
                    self.host_out[b] = host
            self.reps[r].retire(plan, posts, work.local)
        for e in plan.entries:
            self.tags[e.block_index] = (e.noise_level, self.cond.id)
        if timing:
            torch.cuda.synchronize()
            self.rank_times.append([sum(a.elapsed_time(b) for a, b in marks.get(r, []))
                                    for r in range(self.world)])
        self.slot_epoch.wrote([self.slots.slot_of(b) for b in blocks], epoch, items[0][1].masks)
        ev = torch_event(self.torch)
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

    def replica_outputs(self, block):
        """Every rank's emitted copy of `block` (rows partition: all ranks)."""
        self.torch.cuda.current_stream().synchronize()
        return [rep.final[block].cpu().numpy() for rep in self.reps if block in rep.final]

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


def torch_event(torch):
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    return ev
