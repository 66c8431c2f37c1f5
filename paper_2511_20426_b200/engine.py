"""Session loops: the cascaded pipeline and the sequential block-causal
rollout, with the reference signatures (``engine.py:69-342``).

Both loops keep every block's latents and KV on the device:

* the host runs the scheduler (``plan_iteration``/``advance``), the pool
  index logic (``KVPool.insert``), mask construction and the slot table;
* each iteration is ONE device step (:meth:`DeviceRuntime.step`): the
  batched forward of all in-flight entries plus the fused per-entry update
  -- renoise to the next level with counter-keyed noise (p < emit), emit
  (p == emit), or nothing (cache pass: the KV already sits in the block's
  arena slot, inserting it into the pool is bookkeeping);
* emitted blocks are copied device -> host asynchronously; the trace's
  ``wall_clock`` is CUDA-event time between iteration boundaries on the
  launching stream.

Outputs are a pure function of (config minus workers, seeds, prompt
schedule) exactly as in the reference: the worker count only changes the
trace's placement labels.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .config import CascadeConfig
from .core import NoiseStream, embed_prompt
from .denoiser import build_mask, init_model, visible_block_lists
from .errors import ContractViolation, InvalidInputError
from .executor import CostModel, assign_workers, exchanged_kv_frames
from .interactive import CommandQueue, SwitchEvent, SwitchSpec
from .kvpool import KVPool
from .metrics import Trace, TraceEvent
from .scheduler import CascadeState, advance, plan_iteration

DEFAULT_SESSION_SEED = 20260809
DEFAULT_WEIGHT_SEED = 7

POST_RENOISE, POST_EMIT, POST_CACHE = 0, 1, 2


@dataclass
class RunResult:
    outputs: dict
    trace: Trace
    pool: KVPool
    emitted_order: list
    switch_events: list = field(default_factory=list)
    videos: dict = field(default_factory=dict)     # block -> decoded frames (device), with a decoder

    @property
    def iterations(self) -> int:
        return len(self.trace.events)

    def stacked_outputs(self) -> np.ndarray:
        return np.concatenate([self.outputs[k] for k in sorted(self.outputs)])


def _default_weights(config: CascadeConfig, weight_seed: int):
    if config.model == "toy":
        return init_model(weight_seed, config.layers, config.heads,
                          config.latent_dim, config.cond_dim)
    from .wan import WanWeights
    return WanWeights.random(config, weight_seed)


def _runtime_for(weights, config: CascadeConfig):
    if config.model == "toy":
        from .toy import toy_runtime
        return toy_runtime(weights)
    return weights.runtime()


def _switch_table(switches, config: CascadeConfig) -> dict:
    table = {}
    emit = config.schedule().emit_pass
    for spec in switches or ():
        if spec.at_block is not None and not 0 <= spec.at_block < config.num_blocks:
            raise InvalidInputError(
                f"switch block {spec.at_block} outside run of {config.num_blocks} blocks")
        it = spec.boundary_iteration(config.offset, emit)
        if it in table:
            raise InvalidInputError(f"two switches scripted for iteration {it}")
        table[it] = spec
    return table


class _Session:
    """Device-side state of one run shared by both loops."""

    def __init__(self, config, weights, conditioning, session_seed, noise_feed=None):
        self.config = config
        self.rt = _runtime_for(weights, config)
        self.session = self.rt.open_session(config, conditioning, session_seed,
                                            noise_feed=noise_feed)
        self.noise = NoiseStream(session_seed, config.latent_dim)

    def close(self):
        self.session.close()


class _DecodeLane:
    """The reference's decode lane (``engine.py:151-158``: a cost-model charge,
    overlapped on a second worker with ``decode_overlap``) made real: every
    emitted block's x0 is decoded to video frames by a device VAE
    (:class:`~paper_2511_20426_b200.vae.VaeDecoder`) on its own stream, so
    decoding block b overlaps the denoising iterations that follow.  The
    trace's ``decode_start`` / ``decode_done`` get CUDA-event times on the
    same origin as ``wall_clock`` (``metrics.streaming_fps(trace,
    clock="decoded")`` is the paper's decode-inclusive streaming FPS,
    ``PAPER.md:246``)."""

    def __init__(self, decoder, dev, config):
        if config.model != "wan":
            raise InvalidInputError("VAE decode needs the Wan-shaped model (latents (S, 16, h, w))",
                                    fields=["model"])
        import torch
        self.torch = torch
        self.videos, self.marks = {}, []
        self.dev = dev
        # decode on a dedicated GPU (decode_rank.RemoteDecoder): hand every
        # emitted block to the decode rank; its times live on that rank
        self.remote = decoder if getattr(decoder, "remote", False) else None
        if self.remote is not None:
            return
        dc = decoder.cfg
        if (dc.block_size, dc.z_dim, dc.latent_h, dc.latent_w) != (
                config.block_size, config.latent_channels, config.latent_height, config.latent_width):
            raise InvalidInputError("VAE geometry does not match the run's latents", fields=["decoder"])
        self.decoder = decoder
        decoder.reset()

    def emit(self, block, event):
        torch = self.torch
        z = self.dev.emitted_device(block)
        if self.remote is not None:
            self.remote.emit(block, z)
            return
        st = self.decoder.stream
        st.wait_stream(torch.cuda.current_stream())
        z.record_stream(st)                     # the session may free it before the decode ran
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(st)
        self.videos[block] = self.decoder.decode_block(z)
        s1.record(st)
        self.marks.append((event, s0, s1))

    def finish(self):
        if self.remote is not None:
            self.remote.finish()
            return
        self.decoder.stream.synchronize()
        origin = self.dev.events[0]
        for ev, s0, s1 in self.marks:
            ev.decode_start = origin.elapsed_time(s0) / 1e3
            ev.decode_done = origin.elapsed_time(s1) / 1e3
        self.marks.clear()


def _collect_outputs(dev, blocks) -> dict:
    """Emitted blocks as host arrays; multi-GPU sessions gather them from
    their owner ranks."""
    gather = getattr(dev, "gather_outputs", None)
    if gather is not None:
        return gather(list(blocks))
    return {b: dev.emitted_host(b) for b in blocks}


def _recache(dev, pool, targets, S, iteration):
    """KV recache (reference ``kvpool.recache``, kvpool.py:109-140): every
    target pool block, in ascending order, reruns one causal level-0 forward
    from its emitted x0 under the new conditioning, attending to its
    already-recached pool predecessors; its KV is rewritten in place.  Only
    the recache comparison baseline and ``refresh_sink_on_switch`` get here.
    Returns the rebuilt pool and the visible frames of each pass."""
    frames = []
    dev.begin_stall()
    for b in targets:
        preds = [x for x in pool.block_indices if x < b]
        mask = build_mask([b], preds, "causal", S)
        dev.recache_block(b, mask, visible_block_lists(mask)[0])
        pool = pool.insert(b, dev.kv_handle(b))
        frames.append(mask.visible_frames(b))
    dev.end_stall(iteration)
    return pool, frames


def run_cascade(config: CascadeConfig, prompt: str,
                session_seed: int = DEFAULT_SESSION_SEED,
                weight_seed: int = DEFAULT_WEIGHT_SEED,
                switches=(), command_queue: CommandQueue | None = None,
                event_sink=None, weights=None, pace_seconds: float = 0.0,
                noise_feed=None, decoder=None) -> RunResult:
    """Plan / execute / apply until every block has retired (Alg. 1).
    ``decoder`` (a :class:`~paper_2511_20426_b200.vae.VaeDecoder`, optional):
    decode each emitted block on the device, overlapped (``_DecodeLane``)."""
    config.validate()
    if config.decode_overlap and config.workers < 2:
        raise InvalidInputError("decode overlap needs at least 2 workers",
                                fields=["decode_overlap", "workers"])
    sched = config.schedule()
    if weights is None:
        weights = _default_weights(config, weight_seed)
    cond = embed_prompt(prompt, config.cond_dim)
    cost = CostModel.from_config(config)
    pool = KVPool.empty(config.window_blocks, config.sink_blocks)
    state = CascadeState(num_blocks=config.num_blocks, offset=config.offset,
                         schedule=sched, workers=config.workers)
    scripted = _switch_table(switches, config)
    trace = Trace(meta={"kind": "cascade", "prompt": prompt, "session_seed": session_seed,
                        "weight_seed": weight_seed, "config": config.to_dict()})
    sess = _Session(config, weights, cond, session_seed, noise_feed)
    dev = sess.session
    lane = _DecodeLane(decoder, dev, config) if decoder is not None else None
    switch_events = []
    modeled = 0.0
    decode_done_at = 0.0
    pending = []           # (iteration-record) waiting for device timings
    S = config.block_size
    try:
        while not state.done:
            record = None
            spec = scripted.pop(state.iteration, None)
            live = None
            if spec is None and command_queue is not None:
                live = command_queue.pop()
                if live is not None:
                    spec = SwitchSpec(prompt=live.prompt, mode=live.mode,
                                      at_iteration=state.iteration)
            stall = 0.0
            if spec is not None:
                cond = embed_prompt(spec.prompt, config.cond_dim)
                dev.set_conditioning(cond)
                extra = 0
                if spec.mode == "recache":
                    targets = pool.block_indices
                elif config.refresh_sink_on_switch and pool.sink_indices:
                    targets = pool.sink_indices[:1]
                else:
                    targets = ()
                if targets:
                    # comparison baseline only: the product
                    # switch is mode="cascade", which touches no KV
                    pool, frames = _recache(dev, pool, targets, S, state.iteration)
                    extra = len(frames)
                    stall = sum(cost.pass_cost(v) for v in frames)
                ev = SwitchEvent(iteration=state.iteration, boundary_block=state.lead,
                                 mode=spec.mode, extra_passes=extra, conditioning_id=cond.id,
                                 prompt=spec.prompt, stall_modeled=stall)
                switch_events.append(ev)
                record = ev.to_dict()
                if live is not None:
                    live.resolve(ev)

            plan = plan_iteration(state)
            mask = build_mask(plan.blocks, pool.block_indices, config.attention_mode, S)
            pre_pool = pool
            posts = []
            for e in plan.entries:
                if e.pass_index < sched.emit_pass:
                    posts.append((POST_RENOISE, e.pass_index + 1,
                                  sched.level_for_pass(e.pass_index + 1)))
                elif e.pass_index == sched.emit_pass:
                    posts.append((POST_EMIT, None, None))
                else:
                    posts.append((POST_CACHE, None, None))
            dev.step(plan, mask, pool, visible_block_lists(mask), posts)

            emitted = advance(state, plan, plan.blocks)
            for e, (kind, _, _) in zip(plan.entries, posts):
                if kind == POST_CACHE:
                    newer = pool.insert(e.block_index, dev.kv_handle(e.block_index))
                    for gone in pool.evicted_by(newer):
                        dev.release(gone)
                    if e.block_index not in newer:
                        dev.release(e.block_index)
                    pool = newer
            emitted_block = emitted[0] if emitted else None

            # modeled clock: exactly the reference's accounting
            placement = assign_workers(plan.width, config.workers)
            busy = [0.0] * config.workers
            entry_rows = []
            for pos, e in enumerate(plan.entries):
                frames = mask.visible_frames(e.block_index)
                c = cost.pass_cost(frames)
                busy[placement[pos]] += c
                entry_rows.append({"block": e.block_index, "pass_index": e.pass_index,
                                   "noise_level": e.noise_level, "worker": placement[pos],
                                   "conditioning_id": cond.id, "queries": S,
                                   "visible_frames": frames, "modeled_cost": c})
            comm = cost.comm_cost(exchanged_kv_frames(plan.blocks, placement,
                                                      config.attention_mode, S))
            dec_charge = 0.0
            dec_start = dec_done = None
            if emitted_block is not None and cost.decode > 0.0:
                if config.decode_overlap:
                    dec_start = max(modeled + max(busy) + comm, decode_done_at)
                    dec_done = dec_start + cost.decode_cost()
                    decode_done_at = dec_done
                else:
                    dec_charge = cost.decode_cost()
            modeled += stall + max(busy) + comm + dec_charge

            event = TraceEvent(
                iteration=plan.iteration, entries=entry_rows, wall_seconds=0.0,
                modeled_exec=max(busy), modeled_comm=comm, modeled_stall=stall,
                modeled_decode=dec_charge, modeled_clock=modeled, wall_clock=0.0,
                pool_blocks=len(pre_pool.block_indices), pool_frames=pre_pool.frame_count(),
                pool_state=pre_pool.state_dump(), emitted_block=emitted_block,
                emitted_video_frames=(S * config.video_frames_per_latent
                                      if emitted_block is not None else None),
                decode_start=dec_start, decode_done=dec_done, switch=record)
            trace.append(event)
            pending.append(event)
            if lane is not None and emitted_block is not None:
                lane.emit(emitted_block, event)
            if event_sink is not None:
                dev.fill_wall_times(pending)
                pending.clear()
                out = dev.emitted_host(emitted_block) if emitted_block is not None else None
                event_sink(event, out)
            if pace_seconds > 0.0:
                time.sleep(pace_seconds)
        dev.fill_wall_times(pending)
        if lane is not None:
            lane.finish()
        outputs = _collect_outputs(dev, state.emitted)
    finally:
        sess.close()
    if command_queue is not None:
        command_queue.reject_all(InvalidInputError("session already finished"))
    if sorted(outputs) != list(range(config.num_blocks)):
        raise ContractViolation(
            f"run finished with outputs for {sorted(outputs)}; expected all of "
            f"0..{config.num_blocks - 1}")
    return RunResult(outputs=outputs, trace=trace, pool=pool,
                     emitted_order=list(state.emitted), switch_events=switch_events,
                     videos=lane.videos if lane is not None else {})


def run_sequential_reference(config: CascadeConfig, prompt: str,
                             session_seed: int = DEFAULT_SESSION_SEED,
                             weight_seed: int = DEFAULT_WEIGHT_SEED,
                             weights=None, noise_feed=None, decoder=None) -> RunResult:
    """Plain block-causal rollout: every block runs all its passes against
    its predecessors' cached KV before the next block starts.  Written as
    nested loops over (block, pass), independent of the state machine, so
    ``run_cascade(offset=passes)`` can be checked against it."""
    config.validate()
    sched = config.schedule()
    if weights is None:
        weights = _default_weights(config, weight_seed)
    cond = embed_prompt(prompt, config.cond_dim)
    cost = CostModel.from_config(config)
    pool = KVPool.empty(config.window_blocks, config.sink_blocks)
    S = config.block_size
    trace = Trace(meta={"kind": "sequential", "prompt": prompt,
                        "session_seed": session_seed, "weight_seed": weight_seed,
                        "config": config.to_dict()})
    sess = _Session(config, weights, cond, session_seed, noise_feed)
    dev = sess.session
    lane = _DecodeLane(decoder, dev, config) if decoder is not None else None
    emitted_order = []
    modeled = 0.0
    it = 0
    try:
        for b in range(config.num_blocks):
            for p in range(sched.passes):
                level = sched.level_for_pass(p)
                mask = build_mask([b], pool.block_indices, config.attention_mode, S)
                if p < sched.emit_pass:
                    post = (POST_RENOISE, p + 1, sched.level_for_pass(p + 1))
                elif p == sched.emit_pass:
                    post = (POST_EMIT, None, None)
                else:
                    post = (POST_CACHE, None, None)
                from .scheduler import BatchPlan, PlanEntry
                plan = BatchPlan(iteration=it, entries=(PlanEntry(b, p, level, 0),))
                dev.step(plan, mask, pool, visible_block_lists(mask), [post])
                frames = mask.visible_frames(b)
                pc = cost.pass_cost(frames)
                emitted_block = b if p == sched.emit_pass else None
                if emitted_block is not None:
                    emitted_order.append(b)
                pre_pool = pool
                if p == sched.cache_pass:
                    newer = pool.insert(b, dev.kv_handle(b))
                    for gone in pool.evicted_by(newer):
                        dev.release(gone)
                    pool = newer
                dec = cost.decode_cost() if (emitted_block is not None and cost.decode > 0.0) else 0.0
                modeled += pc + dec
                trace.append(TraceEvent(
                    iteration=it,
                    entries=[{"block": b, "pass_index": p, "noise_level": level, "worker": 0,
                              "conditioning_id": cond.id, "queries": S,
                              "visible_frames": frames, "modeled_cost": pc}],
                    wall_seconds=0.0, modeled_exec=pc, modeled_comm=0.0, modeled_stall=0.0,
                    modeled_decode=dec, modeled_clock=modeled, wall_clock=0.0,
                    pool_blocks=len(pre_pool.block_indices),
                    pool_frames=pre_pool.frame_count(), pool_state=pre_pool.state_dump(),
                    emitted_block=emitted_block,
                    emitted_video_frames=(S * config.video_frames_per_latent
                                          if emitted_block is not None else None)))
                if lane is not None and emitted_block is not None:
                    lane.emit(emitted_block, trace.events[-1])
                it += 1
        dev.fill_wall_times(trace.events)
        if lane is not None:
            lane.finish()
        outputs = _collect_outputs(dev, emitted_order)
    finally:
        sess.close()
    return RunResult(outputs=outputs, trace=trace, pool=pool, emitted_order=emitted_order,
                     videos=lane.videos if lane is not None else {})
