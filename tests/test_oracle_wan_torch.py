"""Pin the torch fp32 Wan checker (oracle/wan_torch.py) to the numpy fp32
oracle (oracle/wan.py) and its sub-operators to torch.nn.functional, on CPU.
The torch restatement is what the full-depth GPU parity tests
(tests/test_gpu_wan_full.py) compare the product against, so it must agree
with oracle/wan.py to fp32 round-off before it is trusted there."""

import numpy as np
import pytest
import torch

from oracle import wan as wo
from oracle import wan_torch as wt


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _params(cfg, seed=3):
    from paper_2511_20426_b200.wan import param_shapes
    rng = np.random.default_rng(seed)
    out = {}
    for name, (shape, fan_in, kind) in param_shapes(cfg).items():
        r = rng.standard_normal(shape).astype(np.float32)
        if kind == "w":
            t = r / np.sqrt(fan_in)
        elif kind == "b":
            t = 0.02 * r
        elif kind == "one":
            t = 1.0 + 0.05 * r
        else:
            t = r / np.sqrt(cfg.model_dim)
        out[name] = t.astype(np.float32)
    return out


def test_subops_match_torch_functional():
    g = torch.Generator().manual_seed(0)
    x = torch.randn(64, 256, generator=g) * 3 + 0.5
    w = 1 + 0.05 * torch.randn(256, generator=g)
    with wt.exact_fp32():
        assert torch.allclose(wt.layer_norm(x), torch.nn.functional.layer_norm(x, (256,), eps=1e-6),
                              rtol=0, atol=2e-6)
        assert torch.allclose(wt.rms_norm(x, w), torch.nn.functional.rms_norm(x, (256,), w, eps=1e-6),
                              rtol=0, atol=2e-6)
        assert torch.allclose(wt.gelu_tanh(x), torch.nn.functional.gelu(x, approximate="tanh"),
                              rtol=0, atol=2e-6)
        q = torch.randn(100, 2 * 128, generator=g)
        k = torch.randn(300, 2 * 128, generator=g)
        v = torch.randn(300, 2 * 128, generator=g)
        ref = torch.nn.functional.scaled_dot_product_attention(
            q.view(100, 2, 128).transpose(0, 1), k.view(300, 2, 128).transpose(0, 1),
            v.view(300, 2, 128).transpose(0, 1)).transpose(0, 1).reshape(100, 256)
        out = wt.attention(q, k, v, 2, head_chunk=1, row_chunk=33)
        assert rel(out, ref) < 1e-6
        # and the numpy oracle's attention agrees with both
        assert rel(wo.attention(q.numpy(), k.numpy(), v.numpy(), 2), ref) < 1e-6


def test_rope_and_patch_tables_match_numpy():
    c, s = wo.rope_tables(9, 3, 8, 8)
    tc, ts = wt.rope_tables(9, 3, 8, 8, "cpu")
    # float64 cos/sin: libm vs torch's vectorised kernels differ in the last ulp
    assert np.abs(c - tc.numpy()).max() < 1e-14 and np.abs(s - ts.numpy()).max() < 1e-14
    x = np.random.default_rng(0).standard_normal((3, 16, 16, 16)).astype(np.float32)
    assert np.array_equal(wo.patchify(x), wt.patchify(torch.from_numpy(x)).numpy())
    y = np.random.default_rng(1).standard_normal((3 * 64, 64)).astype(np.float32)
    assert np.array_equal(wo.unpatchify(y, 3, 16, 16), wt.unpatchify(torch.from_numpy(y), 3, 16, 16).numpy())
    assert rel(wt.sinusoid(750.0, 256, "cpu").numpy(), wo.sinusoid(750.0, 256)) < 1e-7


@pytest.mark.parametrize("mode", ["bidirectional", "causal"])
def test_torch_oracle_matches_numpy_oracle(mode):
    import paper_2511_20426_b200 as bc
    from oracle.schedule import visible_blocks
    cfg = bc.wan_config("tiny", total_frames=18)
    p = _params(cfg)
    rng = np.random.default_rng(5)
    T, d = cfg.tokens_per_block, cfg.model_dim
    pool = {b: [(rng.standard_normal((T, d)).astype(np.float32),
                 rng.standard_normal((T, d)).astype(np.float32)) for _ in range(cfg.layers)]
            for b in (0, 1)}
    batch, levels = [2, 3, 4], [250.0, 500.0, 1000.0]
    lat = {b: rng.standard_normal((cfg.block_size, cfg.latent_dim)).astype(np.float32) for b in batch}
    states = rng.standard_normal((cfg.text_len, cfg.text_dim)).astype(np.float32)
    vis = visible_blocks(batch, [0, 1], mode)
    ref = wo.WanOracle(p, cfg).forward([(b, lat[b], lv) for b, lv in zip(batch, levels)],
                                      pool, vis, states)
    out = wt.WanTorchOracle(p, cfg).forward([(b, lat[b], lv) for b, lv in zip(batch, levels)],
                                           pool, vis, states)
    for (x0, kv), (tx0, tkv, v) in zip(ref, out):
        assert rel(tx0.numpy(), x0) < 1e-6
        for l in range(cfg.layers):
            assert rel(tkv[l][0].numpy(), kv[l][0]) < 1e-6
            assert rel(tkv[l][1].numpy(), kv[l][1]) < 1e-6


def test_torch_oracle_session_matches_numpy_session(monkeypatch):
    """The torch oracle session driven by the product engine reproduces the
    numpy oracle session's free-running run (tiny twin, cascade o=1)."""
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import engine
    from oracle.loop import wan_oracle_runtime, wan_torch_oracle_runtime
    cfg = bc.wan_config("tiny", total_frames=12)
    p = _params(cfg)
    with monkeypatch.context() as m:
        m.setattr(engine, "_runtime_for", wan_oracle_runtime(p))
        a = bc.run_cascade(cfg, "a red cube", weights=object())
    with monkeypatch.context() as m:
        m.setattr(engine, "_runtime_for", wan_torch_oracle_runtime(
            {k: torch.from_numpy(v) for k, v in p.items()}))
        b = bc.run_cascade(cfg, "a red cube", weights=object())
    assert a.emitted_order == b.emitted_order
    for k in a.outputs:
        assert rel(b.outputs[k], a.outputs[k]) < 1e-5, k
