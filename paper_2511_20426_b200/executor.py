"""One iteration of the cascade on the device(s).

Reference ``executor.py:27-212`` runs an iteration as fork-join phases over
threads that stand in for GPUs and charges a modeled clock.  Here the whole
batch is one batched device forward per GPU:

* single process / single GPU: ``execute`` calls ``forward`` once for every
  entry of the plan (the width-w batch is one set of kernel launches) and
  times it with CUDA events on the launching stream (``wall_seconds``);
* multi-GPU: :mod:`paper_2511_20426_b200.distributed` splits the batch's
  query rows evenly over the ranks (``rows``, default) or gives whole entries
  to ranks round-robin (``blocks``: ``worker = position % G``, the
  reference's assignment), and hands each layer's fresh K/V to the peers
  with NVLink P2P stores into their IPC-mapped KV arenas plus per-slot
  ready flags, issued by the q/k-norm kernel that produces them (or by a
  side-stream copy, ``BC_KV_PUSH=copy``); torch.distributed (NCCL / gloo)
  carries only the host-side rendezvous and IPC handle exchange.

``CostModel`` and ``exchanged_kv_frames`` are kept with the reference's
arithmetic because the trace schema carries the modeled clock next to the
measured one.
"""

from __future__ import annotations

import contextlib
import time
from dataclasses import dataclass, fields
from typing import NamedTuple

from .errors import ContractViolation, InvalidInputError, IterationError


_COST_FROM_CONFIG = (("pass_base", "pass_cost_base"), ("pass_per_frame", "pass_cost_per_frame"),
                     ("comm_per_frame", "comm_cost_per_frame"), ("decode", "decode_cost"))


@dataclass(frozen=True)
class CostModel:
    """Modeled clock (reference ``executor.py:27-57``), kept because the trace
    carries it next to the measured time: a pass costs ``pass_base +
    pass_per_frame * attended key frames``, a moved KV frame
    ``comm_per_frame``, an emitted block's decode ``decode``."""

    pass_base: float = 1.0
    pass_per_frame: float = 0.0
    comm_per_frame: float = 0.0
    decode: float = 0.0

    def __post_init__(self):
        negative = [f.name for f in fields(self) if getattr(self, f.name) < 0]
        if negative:
            raise InvalidInputError("negative cost parameter(s): " + ", ".join(negative))

    @classmethod
    def from_config(cls, config) -> "CostModel":
        return cls(**{mine: getattr(config, theirs) for mine, theirs in _COST_FROM_CONFIG})

    def pass_cost(self, visible_frames: int) -> float:
        return self.pass_base + visible_frames * self.pass_per_frame

    def comm_cost(self, kv_frames: int) -> float:
        return kv_frames * self.comm_per_frame

    def decode_cost(self) -> float:
        return self.decode


class EntryTiming(NamedTuple):
    block_index: int
    pass_index: int
    worker: int
    visible_frames: int
    modeled_cost: float
    wall_seconds: float


class IterationResult(NamedTuple):
    outputs: list
    timings: list
    modeled_exec: float       # busiest placement, modeled units
    modeled_comm: float
    exchanged_frames: int
    wall_seconds: float       # CUDA-event time of the iteration


class WorkerPool(contextlib.AbstractContextManager):
    """Number of placement slots (GPUs).  The reference's pool is a thread
    pool standing in for GPUs; here a width-w batch is one launch sequence
    per GPU, so ``map`` is a plain in-order loop."""

    def __init__(self, workers: int):
        if not workers >= 1:
            raise InvalidInputError(f"need at least one worker (got {workers})")
        self.workers = workers

    def map(self, fn, items):
        return list(map(fn, items))

    def close(self):
        return None

    def __exit__(self, *exc):
        self.close()


def assign_workers(n_entries: int, workers: int) -> list:
    return [pos % workers for pos in range(n_entries)]


def exchanged_kv_frames(plan_blocks, assignment, mode: str, block_size: int) -> int:
    """KV frames shipped across placements in one iteration: each entry's
    fresh KV goes once to every *other* placement hosting a consumer
    (bidirectional: everyone; causal: higher blocks only)."""
    total = 0
    for i, src in enumerate(plan_blocks):
        targets = {assignment[j] for j, dst in enumerate(plan_blocks)
                   if assignment[j] != assignment[i]
                   and (mode == "bidirectional" or src <= dst)}
        total += block_size * len(targets)
    return total


class _DeviceTimer:
    """CUDA-event wall time of the work launched between start() and stop()
    on the current stream; falls back to perf_counter only for the
    host-array API path (which synchronises anyway)."""

    def __init__(self):
        self._t0 = self._ev0 = self._ev1 = None
        try:
            import torch
            if torch.cuda.is_available():
                self._ev0 = torch.cuda.Event(enable_timing=True)
                self._ev1 = torch.cuda.Event(enable_timing=True)
        except ImportError:  # pragma: no cover
            pass

    def start(self):
        self._t0 = time.perf_counter()
        if self._ev0 is not None:
            self._ev0.record()

    def stop(self) -> float:
        if self._ev1 is not None:
            self._ev1.record()
            self._ev1.synchronize()
            return self._ev0.elapsed_time(self._ev1) / 1e3
        return time.perf_counter() - self._t0


def execute(plan, entries, visible_kv, mask, weights, pool: WorkerPool,
            cost_model: CostModel, mode: str) -> IterationResult:
    """Run one iteration's batch (reference ``executor.py:129-186``).

    Any failure is re-raised as :class:`IterationError` naming the entry
    (the device reports the first offending block through its status flag).
    """
    from . import denoiser

    entries = list(entries)
    if [e.block_index for e in entries] != plan.blocks:
        raise ContractViolation(
            f"entries {[e.block_index for e in entries]} do not match plan {plan.blocks}")
    placement = assign_workers(len(entries), pool.workers)
    timer = _DeviceTimer()
    timer.start()
    try:
        outputs = denoiser.forward(weights, entries, visible_kv, mask)
    except IterationError:
        raise
    except Exception as exc:
        bad = getattr(exc, "block_index", None)
        pos = plan.blocks.index(bad) if bad in plan.blocks else 0
        raise IterationError(
            f"worker {placement[pos]} failed on block {entries[pos].block_index} "
            f"pass {plan.entries[pos].pass_index}: {exc}",
            block_index=entries[pos].block_index,
            pass_index=plan.entries[pos].pass_index) from exc
    wall = timer.stop()

    busy = [0.0] * pool.workers
    timings = []
    for pos, e in enumerate(entries):
        frames = mask.visible_frames(e.block_index)
        cost = cost_model.pass_cost(frames)
        busy[placement[pos]] += cost
        timings.append(EntryTiming(e.block_index, plan.entries[pos].pass_index,
                                   placement[pos], frames, cost, wall / len(entries)))
    moved = exchanged_kv_frames(plan.blocks, placement, mode, mask.block_size)
    return IterationResult(outputs=outputs, timings=timings, modeled_exec=max(busy),
                           modeled_comm=cost_model.comm_cost(moved),
                           exchanged_frames=moved, wall_seconds=wall)


# ---------------------------------------------------------------------------
# Decode stand-in (reference executor.py:189-212).  VAE decode is out of the
# timed path (north_star: "VAE decode is timed separately").
# ---------------------------------------------------------------------------

def make_decode_map(pixel_dim: int, latent_dim: int, frames_per_latent: int, seed: int = 0):
    """Fixed full-column-rank (frames_per_latent * pixel_dim, latent_dim) map,
    Philox-keyed by ``seed ^ 0xDEC0DE`` (same draws as the reference)."""
    import numpy as np
    key = np.uint64(seed ^ 0xDEC0DE)
    shape = (frames_per_latent * pixel_dim, latent_dim)
    mat = np.random.Generator(np.random.Philox(key=key)).standard_normal(shape)
    if np.linalg.matrix_rank(mat) != latent_dim:  # pragma: no cover
        raise ContractViolation(f"decode map of shape {shape} is rank-deficient")
    return mat


def decode_block(latents, decode_map, frames_per_latent: int):
    """(S, D) latents -> (S * frames_per_latent, pixel_dim) frames."""
    rows, width = decode_map.shape if decode_map.ndim == 2 else (-1, -1)
    if width != latents.shape[1] or rows < 0 or rows % frames_per_latent:
        raise ContractViolation(
            f"cannot decode latents {latents.shape} with a map of shape {decode_map.shape}")
    return (latents @ decode_map.T).reshape(latents.shape[0] * frames_per_latent, rows // frames_per_latent)
