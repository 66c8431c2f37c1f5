"""VAE decode on a dedicated GPU.

The paper: "VAE decoding can be moved to a separate GPU to overlap decoding
with next-block denoising" (``PAPER.md:37``); the reference models it as a
second lane of its cost model (``engine.py:151-158``, ``decode_overlap``).
Here it is a real device pipeline: in a job of N processes, ranks 0..N-2 run
the temporal-parallel denoiser (their own process group) and rank N-1 only
decodes.  Each emitted block's x0 (fp32 ``(S, 16, h, w)``, 1.2 MB at
480x832) goes from the emitting denoiser rank straight into an inbox ring in
the decode GPU's memory:

* producer (denoiser rank 0), on a side stream that first waits for the step
  that emitted the block, as handoff item ``k`` (items count on across
  generations; blocks arrive in ascending order): wait until the consumer
  has released inbox slot ``k % R`` (``consumed >= k - R + 1``, a stream
  memory wait on the producer's own flag word), copy the block into the slot
  (a peer copy over NVLink between GPUs: the copy engines, no SM), write
  ``ready = k + 1`` into the consumer's flag word (a stream memory write,
  fenced after the copy);
* consumer (the decode rank), on the decoder's stream: wait ``ready >= k + 1``,
  decode the slot (``VaeDecoder.decode_block``), write ``consumed = k + 1``
  into the producer's flag word.

No SM ever spins: both waits are executed by the streams' front ends
(``cuStreamWaitValue32``), so the protocol is safe even when the two ranks
share one GPU (the two-process test).  Blocks are emitted in ascending
order, so one counter per direction orders everything.  Buffers are CUDA-IPC
memory exchanged once over the world group.
"""

from __future__ import annotations

import ctypes
import time

from . import _native as N
from .errors import ContractViolation, InvalidInputError

INBOX_SLOTS = 4


def split_ranks(decode_gpu: bool):
    """Collective over the world group.  With ``decode_gpu`` the last rank
    becomes the decode rank and the others form the denoiser group
    (installed as :data:`distributed.DIT_GROUP` for ``DistWanSession``).
    Returns ``(is_decode_rank, decode_rank or None)``."""
    import torch.distributed as dist
    from . import distributed
    world, rank = dist.get_world_size(), dist.get_rank()
    if not decode_gpu:
        distributed.DIT_GROUP = None
        return False, None
    if world < 2:
        raise InvalidInputError("a decode GPU needs at least 2 ranks (denoiser + decoder)",
                                fields=["decode_gpu"])
    if world > 2 and distributed.shard_mode() != "rows":
        # checked on every rank (same environment) before any collective, so
        # a misconfigured job fails everywhere instead of hanging
        raise InvalidInputError("a decode GPU needs the rows partition (every denoiser rank "
                                "holds every emitted block)", fields=["BC_TEMPORAL_SHARD"])
    dec = world - 1
    group = dist.new_group(ranks=list(range(dec)))       # every rank must take part
    distributed.DIT_GROUP = group
    return rank == dec, dec


def _ipc_alloc(nbytes):
    ptr = ctypes.c_void_p()
    handle = ctypes.create_string_buffer(64)
    N.check(N.lib().bc_ipc_malloc(int(nbytes), ctypes.byref(ptr), handle), "bc_ipc_malloc")
    return ptr.value, handle.raw


def _ipc_open(handle: bytes):
    ptr = ctypes.c_void_p()
    N.check(N.lib().bc_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(ptr)), "bc_ipc_open")
    return ptr.value


class DecodeHandoff:
    """Both ends of the inbox protocol (module docstring).  Construct it on
    EVERY rank of the world group (it exchanges IPC handles); the producer is
    denoiser rank 0, the consumer the decode rank."""

    def __init__(self, config, decode_rank: int, producer: int = 0, slots: int = INBOX_SLOTS):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank = dist.get_rank()
        self.producer, self.consumer = producer, decode_rank
        self.slots = slots
        self.shape = (config.block_size, config.latent_channels, config.latent_height, config.latent_width)
        self.bytes = 4 * config.block_size * config.latent_channels * config.latent_height * config.latent_width
        self.role = ("producer" if self.rank == producer else
                     "consumer" if self.rank == decode_rank else None)
        self._own, self._opened = [], []
        mine = (self.rank, None, None)
        if self.role == "consumer":
            self.inbox, ih = _ipc_alloc(self.bytes * slots)
            self.flags, fh = _ipc_alloc(64)          # word 0: ready (blocks landed)
            self._own += [self.inbox, self.flags]
            mine = (self.rank, ih, fh)
        elif self.role == "producer":
            self.flags, fh = _ipc_alloc(64)          # word 0: consumed (slots released)
            self._own.append(self.flags)
            mine = (self.rank, None, fh)
        everyone = [None] * dist.get_world_size()
        dist.all_gather_object(everyone, mine)
        if self.role == "producer":
            _, ih, fh = everyone[decode_rank]
            self.peer_inbox, self.peer_flags = _ipc_open(ih), _ipc_open(fh)
            self._opened += [self.peer_inbox, self.peer_flags]
            self.stream = torch.cuda.Stream()
        elif self.role == "consumer":
            _, _, fh = everyone[producer]
            self.peer_flags = _ipc_open(fh)
            self._opened.append(self.peer_flags)
        # handoff sequence numbers run on across generations (the flags are
        # monotonic counters): block k of a run is item seq0 + k
        self.sent = 0      # producer: items handed off so far
        self.served = 0    # consumer: items decoded so far
        self._next_block = 0

    # -- producer ---------------------------------------------------------
    def send(self, block: int, z):
        """Enqueue the handoff of emitted block ``block`` (device fp32 x0 of
        shape (S, 16, h, w)); ordered after the current stream's work.
        Blocks of a run arrive in ascending order from 0."""
        if self.role != "producer":
            return
        if block != 0 and block != self._next_block:
            raise ContractViolation(f"decode handoff expects block {self._next_block}, got {block}")
        self._next_block = block + 1
        torch = self.torch
        if tuple(z.shape) != self.shape or z.dtype != torch.float32 or not z.is_contiguous():
            raise ContractViolation(f"decode handoff: block latents {tuple(z.shape)} {z.dtype}")
        st = self.stream
        st.wait_stream(torch.cuda.current_stream())
        z.record_stream(st)
        sp = N.stream_ptr(st)
        seq = self.sent
        if seq >= self.slots:   # the slot's previous item has been decoded
            N.check(N.lib().bc_stream_wait_geq_u32(self.flags, seq - self.slots + 1, sp), "handoff wait")
        N.check(N.lib().bc_copy_async(self.peer_inbox + (seq % self.slots) * self.bytes, N.ptr(z),
                                      self.bytes, sp), "handoff copy")
        N.check(N.lib().bc_stream_write_u32(self.peer_flags, seq + 1, sp), "handoff ready")
        self.sent += 1

    def flush(self):
        if self.role == "producer":
            self.stream.synchronize()

    # -- consumer ---------------------------------------------------------
    def serve(self, decoder, num_blocks: int, origin=None):
        """Decode blocks 0..num_blocks-1 as they land.  Returns
        ``(videos, times)``: device video tensors per block and, per block,
        ``(decode_start, decode_done)`` seconds after ``origin`` (a CUDA event
        recorded on this rank's current stream; default: now)."""
        if self.role != "consumer":
            raise ContractViolation("serve() runs on the decode rank")
        torch = self.torch
        if origin is None:
            origin = torch.cuda.Event(enable_timing=True)
            origin.record()
        st = decoder.stream
        st.wait_stream(torch.cuda.current_stream())
        sp = N.stream_ptr(st)
        inbox = _raw_f32(self.inbox, (self.slots,) + self.shape)
        videos, marks = {}, []
        decoder.reset()
        for b in range(num_blocks):
            seq = self.served
            N.check(N.lib().bc_stream_wait_geq_u32(self.flags, seq + 1, sp), "decode wait")
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(st)
            with torch.cuda.stream(st):
                videos[b] = decoder.decode_block(inbox[seq % self.slots])
            s1.record(st)
            N.check(N.lib().bc_stream_write_u32(self.peer_flags, seq + 1, sp), "decode release")
            marks.append((s0, s1))
            self.served += 1
        st.synchronize()
        times = [(origin.elapsed_time(s0) / 1e3, origin.elapsed_time(s1) / 1e3) for s0, s1 in marks]
        return videos, times

    def close(self):
        torch = self.torch
        torch.cuda.synchronize()
        self.dist.barrier()
        for p in self._opened:
            N.lib().bc_ipc_close(p)
        for p in self._own:
            N.lib().bc_free(p)
        self._opened, self._own = [], []


def _raw_f32(ptr, shape):
    torch = N.torch_mod()

    class _A:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_A(), device="cuda")


class RemoteDecoder:
    """What a denoiser rank passes as ``run_cascade(decoder=...)`` when the
    decode runs on the decode rank: every emitted block is handed off (by
    denoiser rank 0) instead of decoded locally."""

    remote = True

    def __init__(self, handoff: DecodeHandoff):
        self.handoff = handoff

    def emit(self, block, z):
        self.handoff.send(block, z)

    def finish(self):
        self.handoff.flush()


def decoded_fps(times, frames_per_block: int, blocks=(8, 9)) -> dict:
    """Decode-inclusive FPS on the decode rank's clock: end to end (all
    frames / time the last block finished decoding) and streaming (the paper's
    blocks 8 and 9, 1-indexed: frames per interval between consecutive
    decode completions, ``PAPER.md:246``)."""
    done = [t[1] for t in times]
    out = {"e2e_fps_decoded": len(done) * frames_per_block / done[-1] if done else None}
    rates = [frames_per_block / (done[b - 1] - done[b - 2]) for b in blocks if b - 1 < len(done) and b >= 2]
    out["streaming_fps_decoded"] = sum(rates) / len(rates) if rates else None
    return out


def wall_origin():
    """A host timestamp and a CUDA event recorded together right after a
    barrier: the common origin of a multi-process measurement."""
    import torch
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    return time.monotonic(), ev
