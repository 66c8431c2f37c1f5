"""CPU session runtime for the product engine's session protocol -- TEST
ORACLE ONLY.

``paper_2511_20426_b200.engine`` asks its runtime for a session exposing
``set_conditioning / step / kv_handle / release / emitted_host /
fill_wall_times / close``.  Tests monkeypatch ``engine._runtime_for`` with
:func:`oracle_runtime` to drive the product scheduler / pool / mask / switch
logic on CPU with the numpy oracle forward, and compare against outputs the
reference itself produced (tests/golden).  Never used by the product.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import toy as toy_oracle

POST_RENOISE, POST_EMIT, POST_CACHE = 0, 1, 2


@dataclass(frozen=True)
class _KV:
    block_index: int
    layer_index: int
    keys: np.ndarray
    values: np.ndarray
    noise_tag: float
    conditioning_id: str

    @property
    def frame_count(self):
        return self.keys.shape[0]


class ToyOracleSession:
    def __init__(self, weights, config, cond, session_seed):
        from paper_2511_20426_b200.core import NoiseStream
        self.W = toy_oracle.weights_from(weights)
        self.S = config.block_size
        self.noise = NoiseStream(session_seed, config.latent_dim)
        self.latents, self.final, self.kv, self.tags = {}, {}, {}, {}
        self.cond = cond

    def set_conditioning(self, cond):
        self.cond = cond

    def step(self, plan, mask, pool, vis_lists, posts):
        S = self.S
        ents = []
        for e in plan.entries:
            b = e.block_index
            if e.pass_index == 0 and b not in self.latents:
                self.latents[b] = self.noise.block_noise(b, 0, b * S, S)
            ents.append((b, self.latents[b], e.noise_level, self.cond.embedding))
        visible = {b: lst for b, lst in zip(plan.blocks, vis_lists)}
        pool_kv = {b: self.kv[b] for b in mask.pool_blocks}
        outs = toy_oracle.forward(self.W, ents, pool_kv, visible)
        for e, (x0, kv), (kind, next_pass, next_level) in zip(plan.entries, outs, posts):
            b = e.block_index
            self.kv[b] = kv
            self.tags[b] = (e.noise_level, self.cond.id)
            if kind == POST_RENOISE:
                eps = self.noise.block_noise(b, next_pass, b * S, S)
                self.latents[b] = toy_oracle.renoise(x0, eps, next_level)
            elif kind == POST_EMIT:
                self.final[b] = x0
                self.latents[b] = x0
            else:
                self.latents.pop(b, None)

    def recache_block(self, block, mask, vis_list):
        pool_kv = {b: self.kv[b] for b in mask.pool_blocks}
        (_, kv), = toy_oracle.forward(self.W, [(block, self.final[block], 0.0, self.cond.embedding)],
                                      pool_kv, {block: vis_list})
        self.kv[block] = kv
        self.tags[block] = (0.0, self.cond.id)

    def begin_stall(self):
        pass

    def end_stall(self, iteration):
        pass

    def kv_handle(self, block):
        level, cid = self.tags[block]
        return tuple(_KV(block, l, k, v, level, cid) for l, (k, v) in enumerate(self.kv[block]))

    def release(self, block):
        pass

    def emitted_host(self, block):
        return self.final[block]

    def fill_wall_times(self, events):
        pass

    def close(self):
        pass


class _OracleRuntime:
    def __init__(self, weights):
        self.weights = weights

    def open_session(self, config, cond, session_seed, noise_feed=None):
        return ToyOracleSession(self.weights, config, cond, session_seed)


def oracle_runtime(weights, config):
    """Drop-in replacement for ``engine._runtime_for`` in CPU tests."""
    return _OracleRuntime(weights)


class WanOracleSession:
    """Same protocol, Wan-shaped forward in numpy fp32 (oracle/wan.py)."""

    def __init__(self, params, config, cond, session_seed):
        from paper_2511_20426_b200.core import NoiseStream
        from . import wan as wan_oracle
        self.o = wan_oracle.WanOracle(params, config)
        self.cfg = config
        self.S = config.block_size
        self.shape = (config.block_size, 16, config.latent_height, config.latent_width)
        self.noise = NoiseStream(session_seed, config.latent_dim)
        self.latents, self.final, self.kv, self.tags = {}, {}, {}, {}
        self.set_conditioning(cond)

    def set_conditioning(self, cond):
        from paper_2511_20426_b200.wan import text_states
        self.cond = cond
        self.text_kv = self.o.context(text_states(cond, self.cfg.text_len, self.cfg.text_dim))

    def _noise(self, b, p):
        return self.noise.block_noise(b, p, b * self.S, self.S).astype(np.float32).reshape(self.shape)

    def step(self, plan, mask, pool, vis_lists, posts):
        from . import wan as wan_oracle
        ents = []
        for e in plan.entries:
            b = e.block_index
            if e.pass_index == 0 and b not in self.latents:
                self.latents[b] = self._noise(b, 0)
            ents.append((b, self.latents[b], e.noise_level))
        visible = {b: lst for b, lst in zip(plan.blocks, vis_lists)}
        pool_kv = {b: self.kv[b] for b in mask.pool_blocks}
        outs = self.o.forward(ents, pool_kv, visible, None, text_kv=self.text_kv)
        for e, (x0, kv), (kind, next_pass, next_level) in zip(plan.entries, outs, posts):
            b = e.block_index
            self.kv[b] = kv
            self.tags[b] = (e.noise_level, self.cond.id)
            if kind == POST_RENOISE:
                self.latents[b] = wan_oracle.renoise(x0, self._noise(b, next_pass), next_level)
            elif kind == POST_EMIT:
                self.final[b] = x0
                self.latents[b] = x0
            else:
                self.latents.pop(b, None)

    def recache_block(self, block, mask, vis_list):
        pool_kv = {b: self.kv[b] for b in mask.pool_blocks}
        (_, kv), = self.o.forward([(block, self.final[block], 0.0)], pool_kv, {block: vis_list},
                                  None, text_kv=self.text_kv)
        self.kv[block] = kv
        self.tags[block] = (0.0, self.cond.id)

    def begin_stall(self):
        pass

    def end_stall(self, iteration):
        pass

    def kv_handle(self, block):
        level, cid = self.tags[block]
        return tuple(_KV(block, l, k, v, level, cid) for l, (k, v) in enumerate(self.kv[block]))

    def release(self, block):
        pass

    def emitted_host(self, block):
        return self.final[block].reshape(self.S, -1).astype(np.float64)

    def fill_wall_times(self, events):
        pass

    def close(self):
        pass


class _WanOracleRuntime:
    def __init__(self, params):
        self.params = params

    def open_session(self, config, cond, session_seed, noise_feed=None):
        return WanOracleSession(self.params, config, cond, session_seed)


def wan_oracle_runtime(params):
    """engine._runtime_for replacement bound to fixed host parameters."""
    rt = _WanOracleRuntime(params)
    return lambda weights, config: rt


class WanTorchOracleSession(WanOracleSession):
    """Same protocol with the torch fp32 restatement (oracle/wan_torch.py) on
    the GPU: latents, KV and text K/V stay device tensors in fp32 -- the
    checker for full-depth (30/40-layer) runs at the bench geometry."""

    def __init__(self, tensors, config, cond, session_seed):
        from paper_2511_20426_b200.core import NoiseStream
        from . import wan_torch
        self.o = wan_torch.WanTorchOracle(tensors, config)
        self.cfg = config
        self.S = config.block_size
        self.shape = (config.block_size, 16, config.latent_height, config.latent_width)
        self.noise = NoiseStream(session_seed, config.latent_dim)
        self.latents, self.final, self.kv, self.tags = {}, {}, {}, {}
        self.set_conditioning(cond)

    def _noise(self, b, p):
        import torch
        host = self.noise.block_noise(b, p, b * self.S, self.S).astype(np.float32).reshape(self.shape)
        return torch.from_numpy(host).to(self.o.device)

    def step(self, plan, mask, pool, vis_lists, posts):
        from . import wan_torch
        ents = []
        for e in plan.entries:
            b = e.block_index
            if e.pass_index == 0 and b not in self.latents:
                self.latents[b] = self._noise(b, 0)
            ents.append((b, self.latents[b], e.noise_level))
        visible = {b: lst for b, lst in zip(plan.blocks, vis_lists)}
        pool_kv = {b: self.kv[b] for b in mask.pool_blocks}
        outs = self.o.forward(ents, pool_kv, visible, None, text_kv=self.text_kv)
        for e, (x0, kv, _), (kind, next_pass, next_level) in zip(plan.entries, outs, posts):
            b = e.block_index
            self.kv[b] = kv
            self.tags[b] = (e.noise_level, self.cond.id)
            if kind == POST_RENOISE:
                self.latents[b] = wan_torch.renoise(x0, self._noise(b, next_pass), next_level)
            elif kind == POST_EMIT:
                self.final[b] = x0
                self.latents[b] = x0
            else:
                self.latents.pop(b, None)
        keep = set(mask.pool_blocks) | set(plan.blocks)
        for b in [b for b in self.kv if b not in keep]:
            del self.kv[b]          # evicted: bound the fp32 KV held on the device

    def recache_block(self, block, mask, vis_list):
        pool_kv = {b: self.kv[b] for b in mask.pool_blocks}
        (_, kv, _), = self.o.forward([(block, self.final[block], 0.0)], pool_kv, {block: vis_list},
                                     None, text_kv=self.text_kv)
        self.kv[block] = kv
        self.tags[block] = (0.0, self.cond.id)

    def kv_handle(self, block):
        level, cid = self.tags[block]
        return tuple(_KV(block, l, k, v, level, cid) for l, (k, v) in enumerate(self.kv[block]))

    def emitted_host(self, block):
        return self.final[block].reshape(self.S, -1).double().cpu().numpy()


class _WanTorchOracleRuntime:
    def __init__(self, tensors):
        self.tensors = tensors

    def open_session(self, config, cond, session_seed, noise_feed=None):
        return WanTorchOracleSession(self.tensors, config, cond, session_seed)


def wan_torch_oracle_runtime(tensors):
    """engine._runtime_for replacement: the torch fp32 oracle over the given
    parameter tensors (e.g. ``WanWeights.t``, upcast per use)."""
    rt = _WanTorchOracleRuntime(tensors)
    return lambda weights, config: rt
