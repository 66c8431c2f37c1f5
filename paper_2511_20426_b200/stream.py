"""Trace -> event-stream projection (the reference's SSE event schema).

Same lines, byte for byte, as the reference's ``TraceProjector`` /
``events_from_trace`` (gateway.py:49-132): one ``switch`` line per switch,
one ``metrics`` line per iteration, one ``block`` line per emission (with
the block decoded to pixels by the fixed linear stand-in decoder,
executor.py:189-212), and a final ``done`` line.  The projection carries no
wall-clock fields, so a live stream and a replayed one are identical.  The
session service that serves these lines over SSE, fed by the device
engine's ``event_sink``, is :mod:`paper_2511_20426_b200.service`.
"""

from __future__ import annotations

import base64
import json

import numpy as np

from .engine import DEFAULT_WEIGHT_SEED
from .errors import ContractViolation
from .executor import decode_block, make_decode_map


def encode_pixels(pixels: np.ndarray) -> dict:
    """gateway.py:36-42"""
    data = np.ascontiguousarray(pixels, dtype="<f4")
    return {"data": base64.b64encode(data.tobytes()).decode("ascii"),
            "shape": list(data.shape), "dtype": "float32"}


def dumps(doc: dict) -> str:
    """gateway.py:45-46: sorted keys, compact separators."""
    return json.dumps(doc, sort_keys=True, separators=(",", ":"))


class TraceProjector:
    """Incremental projection: feed trace events (and the emitted latents)
    in order, get that iteration's event lines (gateway.py:49-120)."""

    def __init__(self, config, weight_seed: int = DEFAULT_WEIGHT_SEED):
        self.config = config
        self.decode_map = make_decode_map(config.pixel_dim, config.latent_dim,
                                          config.video_frames_per_latent, seed=weight_seed)
        self.seq = 0
        self.last_emission_clock = 0.0
        self.blocks_emitted = 0

    def _next_seq(self) -> int:
        self.seq += 1
        return self.seq - 1

    def feed(self, event, emitted_latents) -> list:
        lines = []
        if event.switch is not None:
            lines.append(dumps({"type": "switch", "seq": self._next_seq(), **event.switch}))
        lines.append(dumps({
            "type": "metrics", "seq": self._next_seq(), "iteration": event.iteration,
            "entries": event.entries, "modeled_exec": event.modeled_exec,
            "modeled_comm": event.modeled_comm, "modeled_stall": event.modeled_stall,
            "modeled_clock": event.modeled_clock, "pool_blocks": event.pool_blocks,
            "pool_frames": event.pool_frames, "phase_width": len(event.entries)}))
        if event.emitted_block is not None:
            if emitted_latents is None:
                raise ContractViolation("emission event without latents")
            elapsed = event.modeled_clock - self.last_emission_clock
            self.last_emission_clock = event.modeled_clock
            pixels = decode_block(np.asarray(emitted_latents, dtype=np.float64), self.decode_map,
                                  self.config.video_frames_per_latent)
            self.blocks_emitted += 1
            lines.append(dumps({
                "type": "block", "seq": self._next_seq(), "index": event.emitted_block,
                "video_frames": event.emitted_video_frames, "elapsed": elapsed,
                "fps": event.emitted_video_frames / elapsed, "pixels": encode_pixels(pixels)}))
        return lines

    def finish(self, trace) -> str:
        return dumps({"type": "done", "seq": self._next_seq(), "blocks": self.blocks_emitted,
                      "iterations": len(trace.events),
                      "total_modeled_time": trace.total_modeled_time,
                      "total_passes": trace.total_passes})


def events_from_trace(trace, config, outputs: dict, weight_seed: int = DEFAULT_WEIGHT_SEED) -> list:
    """Replay path: the whole stream of a finished run (gateway.py:123-132)."""
    proj = TraceProjector(config, weight_seed=weight_seed)
    lines = []
    for ev in trace.events:
        lat = outputs.get(ev.emitted_block) if ev.emitted_block is not None else None
        lines.extend(proj.feed(ev, lat))
    lines.append(proj.finish(trace))
    return lines
