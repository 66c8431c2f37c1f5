"""Shared value types: timestep schedules, prompt conditioning, latent blocks
and the counter-keyed Gaussian noise stream.

Semantics follow the reference ``core.py`` (``TimestepSchedule`` 26-56,
``make_schedule`` 59-73, ``Block`` 91-120, ``embed_prompt`` 144-158,
``NoiseStream`` 161-186).  The noise stream is keyed exactly like the
reference -- numpy's Philox4x64-10 with ``key = session_seed`` and
``counter = [block, pass, frame, 0]`` feeding numpy's ziggurat normal -- so
draws are bit-identical.  Large (Wan-sized) block draws go through the native
multi-threaded generator in ``csrc/noise.cpp`` (same bit generator, numpy's
own ``random_standard_normal_fill`` linked from ``libnpyrandom.a``), which
releases the GIL and writes fp32 straight into pinned host memory.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidInputError

MAX_LEVEL = 1000.0
_U64 = 0xFFFFFFFFFFFFFFFF


def _readonly(arr) -> np.ndarray:
    out = np.array(arr, dtype=np.float64, copy=True, order="C")
    out.flags.writeable = False
    return out


# --------------------------------------------------------------------------
# Counter-keyed noise (reference core.py:161-190)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class NoiseStream:
    """Gaussian draws that are a pure function of (seed, block, pass, frame)."""

    session_seed: int
    dim: int

    def _check(self, *idx):
        if min(idx) < 0:
            raise InvalidInputError("noise stream indices must be >= 0")

    def draw(self, block_index: int, pass_index: int, frame_index: int) -> np.ndarray:
        self._check(block_index, pass_index, frame_index)
        gen = np.random.Generator(np.random.Philox(
            key=np.uint64(self.session_seed & _U64),
            counter=np.array([block_index, pass_index, frame_index, 0], dtype=np.uint64)))
        return gen.standard_normal(self.dim)

    def block_noise(self, block_index: int, pass_index: int, frame0: int, size: int) -> np.ndarray:
        """(size, dim) float64 stack, frames ``frame0 .. frame0+size-1``."""
        self._check(block_index, pass_index, frame0)
        if self.dim * size >= 1 << 16:
            from . import _native
            out = np.empty((size, self.dim), dtype=np.float64)
            _native.noise_block_f64(self.session_seed, block_index, pass_index,
                                    frame0, size, self.dim, out)
            return out
        return np.stack([self.draw(block_index, pass_index, frame0 + i)
                         for i in range(size)])

    def block_noise_f32(self, block_index: int, pass_index: int, frame0: int,
                        size: int, out: np.ndarray | None = None) -> np.ndarray:
        """Same draws rounded to float32 (device latents are fp32), produced
        by the native generator with one thread per frame chunk."""
        self._check(block_index, pass_index, frame0)
        from . import _native
        if out is None:
            out = np.empty((size, self.dim), dtype=np.float32)
        _native.noise_block_f32(self.session_seed, block_index, pass_index,
                                frame0, size, self.dim, out)
        return out


def noise_draw(stream: NoiseStream, block_index: int, pass_index: int,
               frame_index: int) -> np.ndarray:
    return stream.draw(block_index, pass_index, frame_index)


# --------------------------------------------------------------------------
# Conditioning (reference core.py:131-158)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Conditioning:
    """Hash-expanded prompt embedding.  ``id`` is the first 16 hex chars of
    sha256(prompt); ``digest`` keeps the full hash for derived expansions
    (the synthetic text-encoder states of the Wan-shaped model)."""

    prompt: str
    embedding: np.ndarray
    id: str
    digest: bytes = field(default=b"", compare=False, repr=False)

    def __post_init__(self):
        object.__setattr__(self, "embedding", _readonly(self.embedding))

    def key_words(self) -> np.ndarray:
        return np.frombuffer(self.digest[:16], dtype=np.uint64).copy()


def embed_prompt(prompt: str, cond_dim: int) -> Conditioning:
    """sha256(prompt) keys a Philox stream; the embedding is its first
    ``cond_dim`` normals scaled to unit length."""
    if not (isinstance(prompt, str) and prompt):
        raise InvalidInputError("the prompt must be a non-empty str")
    if cond_dim < 1:
        raise InvalidInputError(f"cond_dim {cond_dim} < 1")
    digest = hashlib.sha256(prompt.encode("utf-8")).digest()
    rng = np.random.Generator(np.random.Philox(key=np.frombuffer(digest[:16], dtype=np.uint64)))
    raw = rng.standard_normal(cond_dim)
    return Conditioning(prompt=prompt, embedding=raw / np.linalg.norm(raw), id=digest.hex()[:16], digest=digest)


# --------------------------------------------------------------------------
# Timestep schedule (reference core.py:26-73)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class TimestepSchedule:
    """Denoise levels (strictly decreasing, in (0, 1000]) followed by one
    zero-noise cache pass whose KV is what later blocks attend to."""

    denoise_levels: tuple
    cache_level: float = 0.0

    @property
    def passes(self) -> int:
        return len(self.denoise_levels) + 1

    @property
    def emit_pass(self) -> int:
        # x0 of the last denoise pass is the block's output
        return len(self.denoise_levels) - 1

    @property
    def cache_pass(self) -> int:
        return len(self.denoise_levels)

    def level_for_pass(self, pass_index: int) -> float:
        n = len(self.denoise_levels)
        if 0 <= pass_index < n:
            return self.denoise_levels[pass_index]
        if pass_index == n:
            return self.cache_level
        raise InvalidInputError(
            f"pass index {pass_index} out of range for {self.passes} passes")

    def table(self) -> list:
        """The per-pass level table ``[level(0), ..., level(P-1)]``."""
        return [self.level_for_pass(p) for p in range(self.passes)]


def make_schedule(levels) -> TimestepSchedule:
    """Validate and freeze a denoise-level list: finite, strictly
    decreasing, inside (0, MAX_LEVEL]."""
    vals = tuple(map(float, levels))
    problems = []
    if not vals:
        problems.append("no denoise level given")
    elif not all(map(math.isfinite, vals)):
        problems.append("non-finite level")
    else:
        if vals[0] > MAX_LEVEL or vals[-1] <= 0.0:
            problems.append(f"levels outside (0, {MAX_LEVEL:g}]")
        if any(b >= a for a, b in zip(vals, vals[1:])):
            problems.append("levels not strictly decreasing")
    if problems:
        raise InvalidInputError(f"bad timestep schedule {list(vals)}: " + "; ".join(problems))
    return TimestepSchedule(denoise_levels=vals)


# --------------------------------------------------------------------------
# Latent frames / blocks (reference core.py:76-128)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class LatentFrame:
    frame_index: int
    values: np.ndarray
    noise_level: float

    def __post_init__(self):
        vals = _readonly(self.values)
        if not np.isfinite(vals).all():
            raise InvalidInputError(f"frame {self.frame_index} has non-finite values")
        object.__setattr__(self, "values", vals)


@dataclass(frozen=True)
class Block:
    block_index: int
    frames: tuple
    pass_index: int = 0
    conditioning_id: str = ""

    def __post_init__(self):
        size = len(self.frames)
        want = range(self.block_index * size, (self.block_index + 1) * size)
        got = [fr.frame_index for fr in self.frames]
        if got != list(want):
            raise InvalidInputError(f"block {self.block_index}: frame indices {got}, expected {list(want)}")
        levels = sorted({fr.noise_level for fr in self.frames})
        if len(levels) > 1:
            raise InvalidInputError(f"block {self.block_index}: frames at different noise levels {levels}")

    @property
    def noise_level(self) -> float:
        return self.frames[0].noise_level

    @property
    def latents(self) -> np.ndarray:
        return np.stack([f.values for f in self.frames])


def block_from_latents(block_index, latents, noise_level, conditioning_id="") -> Block:
    n = latents.shape[0]
    return Block(block_index,
                 tuple(LatentFrame(block_index * n + i, latents[i], noise_level)
                       for i in range(n)),
                 conditioning_id=conditioning_id)
