"""Global shared KV pool: index logic on the host, payload in a device arena.

Index semantics are the reference's (``kvpool.py:18-87``): overwrite-insert,
then evict the lowest-indexed non-sink block while more than ``window``
non-sink blocks are held; the sink is block 0 when ``sink_blocks == 1``;
``visible_set(b)`` returns strict predecessors ascending.  A pool is an
immutable value -- every insert returns a new pool -- so an iteration's
snapshot cannot change under it.

The payload per block is whatever the forward produced for it: a tuple of
``LayerKV`` with host arrays (toy model / tests) or a :class:`SlotKV` handle
naming a slot of the device KV arena (every GPU forward).  On the device a
block's slot is written in place by every pass; the cache pass makes it the
pool entry, so inserting is pure bookkeeping -- no copy.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ContractViolation


def _tag_block(kv_layers) -> int:
    return kv_layers[0].block_index


@dataclass(frozen=True)
class KVPool:
    window: int
    sink_blocks: int
    entries: tuple = ()        # ((block, kv_layers), ...) ascending by block

    @classmethod
    def empty(cls, window: int, sink_blocks: int) -> "KVPool":
        return cls(window=window, sink_blocks=sink_blocks)

    def _is_sink(self, block: int) -> bool:
        return block == 0 and self.sink_blocks > 0

    @property
    def block_indices(self) -> list:
        return [b for b, _ in self.entries]

    @property
    def sink_indices(self) -> list:
        return [b for b, _ in self.entries if self._is_sink(b)]

    def get(self, block_index: int):
        for b, kv in self.entries:
            if b == block_index:
                return kv
        raise KeyError(block_index)

    def __contains__(self, block_index) -> bool:
        return any(b == block_index for b, _ in self.entries)

    def insert(self, block_index: int, kv_layers) -> "KVPool":
        kv_layers = kv_layers if isinstance(kv_layers, SlotKV) else tuple(kv_layers)
        tags = {kv.block_index for kv in kv_layers}
        if tags != {block_index}:
            raise ContractViolation(
                f"KV tagged for blocks {sorted(tags)} inserted under block {block_index}")
        held = dict(self.entries)
        held[block_index] = kv_layers
        order = sorted(held)
        regular = [b for b in order if not self._is_sink(b)]
        excess = len(regular) - self.window
        for victim in regular[:max(0, excess)]:
            del held[victim]
        return KVPool(window=self.window, sink_blocks=self.sink_blocks,
                      entries=tuple((b, held[b]) for b in sorted(held)))

    def evicted_by(self, newer: "KVPool") -> list:
        """Blocks held here but not in ``newer`` (slots to release)."""
        keep = set(newer.block_indices)
        return [b for b in self.block_indices if b not in keep]

    def visible_set(self, querying_block: int) -> list:
        return [kv for b, kv in self.entries if b < querying_block]

    def frame_count(self) -> int:
        return sum(kv[0].frame_count for _, kv in self.entries)

    def state_dump(self) -> list:
        return [{"block": b, "noise_tag": kv[0].noise_tag,
                 "conditioning_id": kv[0].conditioning_id, "sink": self._is_sink(b)}
                for b, kv in self.entries]


def insert(pool: KVPool, block_index: int, kv_layers) -> KVPool:
    return pool.insert(block_index, kv_layers)


def visible_set(pool: KVPool, querying_block: int) -> list:
    return pool.visible_set(querying_block)


def pool_frame_count(pool: KVPool) -> int:
    return pool.frame_count()


# ---------------------------------------------------------------------------
# Device-resident KV handles
# ---------------------------------------------------------------------------

class SlotLayerKV:
    """``LayerKV``-compatible view of one layer of one arena slot.  ``keys``
    and ``values`` are materialised (device -> host) only when read."""

    __slots__ = ("block_index", "layer_index", "noise_tag", "conditioning_id",
                 "_arena", "_slot", "frame_count")

    def __init__(self, arena, slot, block_index, layer_index, noise_tag,
                 conditioning_id, frame_count):
        self._arena = arena
        self._slot = slot
        self.block_index = block_index
        self.layer_index = layer_index
        self.noise_tag = noise_tag
        self.conditioning_id = conditioning_id
        self.frame_count = frame_count

    @property
    def keys(self):
        return self._arena.read(self._slot, self.layer_index, which=0)

    @property
    def values(self):
        return self._arena.read(self._slot, self.layer_index, which=1)


class SlotKV:
    """Per-layer KV of one block living in slot ``slot`` of a device arena.
    Behaves like the reference's ``tuple[LayerKV, ...]``."""

    def __init__(self, arena, slot: int, block_index: int, noise_tag: float,
                 conditioning_id: str, frame_count: int):
        self.arena = arena
        self.slot = slot
        self._layers = tuple(
            SlotLayerKV(arena, slot, block_index, layer, noise_tag, conditioning_id,
                        frame_count)
            for layer in range(arena.layers))

    def __len__(self):
        return len(self._layers)

    def __getitem__(self, i):
        return self._layers[i]

    def __iter__(self):
        return iter(self._layers)


class SlotAllocator:
    """Free list over arena slots.  A slot is owned by one block from its
    admission until it leaves the pool (evicted) or the run ends."""

    def __init__(self, n_slots: int):
        self._free = list(range(n_slots - 1, -1, -1))
        self.owner = {}

    def acquire(self, block: int) -> int:
        if block in self.owner:
            return self.owner[block]
        if not self._free:
            raise ContractViolation("KV arena exhausted: no free slot")
        slot = self._free.pop()
        self.owner[block] = slot
        return slot

    def release(self, block: int) -> None:
        slot = self.owner.pop(block, None)
        if slot is not None:
            self._free.append(slot)

    def slot_of(self, block: int) -> int:
        return self.owner[block]


# ---------------------------------------------------------------------------
# Recache (reference kvpool.py:103-140).  Not on the cascade path -- the
# cascade-mode prompt switch never rebuilds KV -- kept so the LongLive-style
# baseline can be measured through the same forward.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class RecacheResult:
    pool: KVPool
    passes: int
    visible_frames: tuple


def recache(pool: KVPool, new_conditioning, weights, block_latents: dict) -> RecacheResult:
    from . import denoiser

    rebuilt = pool
    frames = []
    for b in pool.block_indices:
        if b not in block_latents:
            raise ContractViolation(f"recache needs clean latents for pool block {b}")
        ctx = rebuilt.visible_set(b)
        size = block_latents[b].shape[0]
        mask = denoiser.build_mask([b], [kv[0].block_index for kv in ctx], "causal", size)
        entry = denoiser.EntryInput(block_index=b, latents=block_latents[b],
                                    noise_level=0.0, conditioning=new_conditioning)
        out = denoiser.forward(weights, [entry], ctx, mask)[0]
        rebuilt = rebuilt.insert(b, out.kv)
        frames.append(mask.visible_frames(b))
    return RecacheResult(pool=rebuilt, passes=len(frames), visible_frames=tuple(frames))
