"""The numeric operator boundary: ``forward``, ``renoise``, ``build_mask`` and
the model types, behind the reference signatures (``denoiser.py:29-368``).

Everything numeric runs on the GPU through ``libbcb200.so`` (C-ABI,
``include/bcb200.h``); this module validates arguments exactly like the
reference, maps pool/batch blocks onto device KV-arena slots and dispatches
on the model family:

* :class:`ModelWeights` -- the reference's toy DiT (one token per latent
  frame, float64).  Weights are drawn with the reference's Philox recipe so
  both sides hold identical values; the GPU forward runs in float64.
* :class:`~paper_2511_20426_b200.wan.WanWeights` -- the Wan2.1-shaped DiT
  (bf16 tcgen05 GEMMs + flash attention); see ``wan.py``.

There is no CPU fallback: without a CUDA device the native library refuses
to run and a :class:`~paper_2511_20426_b200.errors.DeviceError` is raised.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .core import MAX_LEVEL, Conditioning
from .errors import ContractViolation, InvalidInputError, NumericError

LEVEL_FEATS = 8
RMS_EPS = 1e-6


# ---------------------------------------------------------------------------
# Toy model weights (reference denoiser.py:29-120)
# ---------------------------------------------------------------------------

@dataclass(frozen=True, eq=False)
class ModelWeights:
    seed: int
    layers: int
    heads: int
    latent_dim: int
    cond_dim: int
    w_in: np.ndarray
    w_cond: np.ndarray
    w_level: np.ndarray
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray
    w_head: np.ndarray

    @property
    def head_dim(self) -> int:
        return self.latent_dim // self.heads

    def arrays(self):
        return (self.w_in, self.w_cond, self.w_level, self.w_q, self.w_k,
                self.w_v, self.w_o, self.w_head)


def _weight_shapes(layers, d, dc):
    return [("w_in", (d, d), d), ("w_cond", (d, dc), dc),
            ("w_level", (d, LEVEL_FEATS), LEVEL_FEATS),
            ("w_q", (layers, d, d), d), ("w_k", (layers, d, d), d),
            ("w_v", (layers, d, d), d), ("w_o", (layers, d, d), d),
            ("w_head", (d, d), d)]


def init_model(weight_seed: int, layers: int, heads: int, latent_dim: int,
               cond_dim: int) -> ModelWeights:
    """Fixed random weights: one Philox(key=seed) stream, N(0,1)/sqrt(fan_in),
    drawn in declaration order -- identical values to the reference."""
    if min(layers, heads, latent_dim, cond_dim) < 1:
        raise InvalidInputError("model dims must all be >= 1")
    if latent_dim % heads:
        raise InvalidInputError(f"heads ({heads}) must divide latent_dim ({latent_dim})")
    gen = np.random.Generator(np.random.Philox(key=np.uint64(weight_seed & 0xFFFFFFFFFFFFFFFF)))
    drawn = {name: gen.standard_normal(shape) / np.sqrt(fan_in)
             for name, shape, fan_in in _weight_shapes(layers, latent_dim, cond_dim)}
    return ModelWeights(seed=weight_seed, layers=layers, heads=heads,
                        latent_dim=latent_dim, cond_dim=cond_dim, **drawn)


_SNAP_HEAD = "<4sIqIIII"
_SNAP_MAGIC = b"BCWT"


def save_weights(weights: ModelWeights, path) -> None:
    """Flat binary snapshot, byte-compatible with the reference format."""
    with open(path, "wb") as fh:
        fh.write(struct.pack(_SNAP_HEAD, _SNAP_MAGIC, 1, weights.seed, weights.layers,
                             weights.heads, weights.latent_dim, weights.cond_dim))
        for arr in weights.arrays():
            fh.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())


def load_weights(path) -> ModelWeights:
    size = struct.calcsize(_SNAP_HEAD)
    with open(path, "rb") as fh:
        head = fh.read(size)
        if len(head) != size or head[:4] != _SNAP_MAGIC:
            raise InvalidInputError(f"{path} is not a weight snapshot")
        _, version, seed, layers, heads, d, dc = struct.unpack(_SNAP_HEAD, head)
        if version != 1:
            raise InvalidInputError(f"{path} is not a weight snapshot")
        arrays = {}
        for name, shape, _ in _weight_shapes(layers, d, dc):
            n = int(np.prod(shape))
            buf = fh.read(n * 8)
            if len(buf) != n * 8:
                raise InvalidInputError(f"truncated weight snapshot {path}")
            arrays[name] = np.frombuffer(buf, dtype="<f8").reshape(shape).copy()
    return ModelWeights(seed, layers, heads, d, dc, **arrays)


# ---------------------------------------------------------------------------
# KV and masks (reference denoiser.py:123-194)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LayerKV:
    block_index: int
    layer_index: int
    keys: np.ndarray
    values: np.ndarray
    noise_tag: float
    conditioning_id: str

    @property
    def frame_count(self) -> int:
        return self.keys.shape[0]


@dataclass(frozen=True)
class AttentionMask:
    """Visibility over (query frame, key frame).  Rows: batch frames in block
    order; columns: pool frames then batch frames, each in block order."""

    batch_blocks: tuple
    pool_blocks: tuple
    block_size: int
    matrix: np.ndarray

    @property
    def key_blocks(self) -> tuple:
        return self.pool_blocks + self.batch_blocks

    def visible_key_blocks(self, query_block: int) -> list:
        row = self.matrix[self.batch_blocks.index(query_block) * self.block_size]
        s = self.block_size
        return sorted(kb for j, kb in enumerate(self.key_blocks) if row[j * s])

    def visible_frames(self, query_block: int) -> int:
        return len(self.visible_key_blocks(query_block)) * self.block_size


def _block_visible(mode: str, key_block: int, query_block: int) -> bool:
    return mode == "bidirectional" or key_block <= query_block


def build_mask(batch_blocks, pool_blocks, mode: str, block_size: int) -> AttentionMask:
    batch = tuple(sorted(int(b) for b in batch_blocks))
    pool = tuple(sorted(int(b) for b in pool_blocks))
    if not batch:
        raise ContractViolation("batch must be non-empty")
    clash = sorted(set(batch) & set(pool))
    if clash:
        raise ContractViolation(f"pool and batch overlap: {clash}")
    if mode not in ("causal", "bidirectional"):
        raise InvalidInputError(f"unknown attention mode {mode!r}")
    keys = pool + batch
    blk = np.array([[_block_visible(mode, kb, qb) for kb in keys] for qb in batch],
                   dtype=bool)
    # expand block visibility to frames: within a block always full
    matrix = np.kron(blk, np.ones((block_size, block_size), dtype=bool))
    matrix.flags.writeable = False
    return AttentionMask(batch_blocks=batch, pool_blocks=pool,
                         block_size=block_size, matrix=matrix)


def visible_block_lists(mask: AttentionMask) -> list:
    """Per batch block (mask order): the visible key blocks, ascending --
    the gather order of reference ``_gather`` (denoiser.py:284-296).  This is
    what the device attention kernels consume as their slot table."""
    return [mask.visible_key_blocks(b) for b in mask.batch_blocks]


# ---------------------------------------------------------------------------
# Entries
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class EntryInput:
    block_index: int
    latents: object              # (S, D) numpy float64, or a device tensor
    noise_level: float
    conditioning: Conditioning


@dataclass(frozen=True)
class EntryOutput:
    block_index: int
    x0: object                   # same container kind as the input latents
    kv: tuple                    # one LayerKV per layer, or a SlotKV handle


def _is_device_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _check_entries(weights, batch, mask, visible_kv):
    if [e.block_index for e in batch] != list(mask.batch_blocks):
        raise ContractViolation(
            f"mask batch {mask.batch_blocks} does not match entries "
            f"{[e.block_index for e in batch]}")
    by_block = {}
    for kv_layers in visible_kv:
        if len(kv_layers) != weights.layers:
            raise ContractViolation(
                f"pool entry for block {kv_layers[0].block_index} has "
                f"{len(kv_layers)} layers, model has {weights.layers}")
        by_block[kv_layers[0].block_index] = kv_layers
    if set(by_block) != set(mask.pool_blocks):
        raise ContractViolation(
            f"mask pool {mask.pool_blocks} does not match supplied KV {sorted(by_block)}")
    for e in batch:
        if e.latents.shape[0] != mask.block_size:
            raise ContractViolation("entry frame count does not match mask block size")
        if not 0.0 <= e.noise_level <= MAX_LEVEL:
            raise ContractViolation(
                f"noise level {e.noise_level} out of [0, {MAX_LEVEL:g}]")
    return by_block


def forward(weights, batch, visible_kv, mask: AttentionMask, mapper=map):
    """Run every batch entry through the layer stack with shared attention.

    Same contract as reference ``forward`` (denoiser.py:299-357).  ``mapper``
    is accepted for signature compatibility and ignored: the fan-out over
    entries happens inside the batched device kernels.
    """
    batch = list(batch)
    pool_kv = _check_entries(weights, batch, mask, visible_kv)
    if isinstance(weights, ModelWeights):
        for e in batch:
            if e.latents.shape[1] != weights.latent_dim:
                raise ContractViolation(
                    f"latents dim {e.latents.shape[1]} does not match model dim "
                    f"{weights.latent_dim}")
        from .toy import toy_runtime
        return toy_runtime(weights).forward(batch, pool_kv, mask)
    from .wan import WanWeights
    if isinstance(weights, WanWeights):
        return weights.runtime().forward(batch, pool_kv, mask)
    raise ContractViolation(f"unsupported weights type {type(weights).__name__}")


def renoise(x0, eps, level: float):
    """(1 - s) * x0 + s * eps with s = level / 1000 (reference
    denoiser.py:360-368), computed by the ``bc_renoise`` device kernel.
    Device tensors stay on the device; host arrays round-trip through it."""
    if tuple(x0.shape) != tuple(eps.shape):
        raise ContractViolation(f"renoise shape mismatch {tuple(x0.shape)} vs {tuple(eps.shape)}")
    if not 0.0 <= level <= MAX_LEVEL:
        raise ContractViolation(f"renoise level {level} out of [0, {MAX_LEVEL:g}]")
    from . import _native
    return _native.renoise(x0, eps, float(level))


def check_finite_host(latents, block_index):
    """Host-side finiteness check used when latents arrive as host arrays
    (the device path checks inside the embedding kernel)."""
    if not np.isfinite(np.asarray(latents)).all():
        raise NumericError(f"non-finite latents in block {block_index}")
