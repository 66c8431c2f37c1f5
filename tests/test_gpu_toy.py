"""Toy DiT on the GPU (float64 kernels, csrc/toy.cu) vs the reference's own
outputs (golden vectors) and the reference's acceptance properties.

Tolerance: the reference computes in float64 with BLAS summation order; the
device computes in float64 with its own fixed order, so agreement is to
~1e-12 relative (stated per assertion).  Equalities between two device runs
(P1 equivalence, worker independence, causal truncation) are exact.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL = 1e-10


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _stack(run):
    return np.stack([run.outputs[k] for k in sorted(run.outputs)])


def test_native_renoise_identities():
    from paper_2511_20426_b200 import renoise
    rng = np.random.default_rng(0)
    x0, eps = rng.standard_normal((3, 4096)), rng.standard_normal((3, 4096))
    assert np.array_equal(renoise(x0, eps, 0.0), x0)
    assert np.array_equal(renoise(x0, eps, 1000.0), eps)
    for lv in (750.0, 333.0, 1.0):
        s = lv / 1000.0
        assert np.array_equal(renoise(x0, eps, lv), (1.0 - s) * x0 + s * eps)


def test_native_renoise_golden(golden):
    from paper_2511_20426_b200 import renoise
    assert np.array_equal(renoise(golden["renoise_x0"], golden["renoise_eps"], 750.0),
                          golden["renoise_750"])


@pytest.mark.parametrize("name", ["small_bidir", "small_causal", "tiny_bidir5",
                                  "tiny_causal5", "tiny_single"])
def test_toy_forward_matches_reference(golden, name):
    import paper_2511_20426_b200 as bc
    c = {k[len(f"case_{name}_"):]: v for k, v in golden.items() if k.startswith(f"case_{name}_")}
    w = bc.init_model(11, 2, 2, 16, 16) if name.startswith("small") else bc.init_model(7, 4, 2, 256, 256)
    cond = bc.embed_prompt(str(c["prompt"]), w.cond_dim)
    batch = [int(b) for b in c["batch"]]
    pool = [int(b) for b in c["pool"]]
    pool_kv = [tuple(bc.LayerKV(b, l, c["pool_k"][i][l], c["pool_v"][i][l], 0.0, cond.id)
                     for l in range(w.layers)) for i, b in enumerate(pool)]
    ents = [bc.EntryInput(b, c["latents"][i], float(c["levels"][i]), cond)
            for i, b in enumerate(batch)]
    mask = bc.build_mask(batch, pool, str(c["mode"]), 3)
    outs = bc.forward(w, ents, pool_kv, mask)
    for i, o in enumerate(outs):
        assert _rel(o.x0, c["x0"][i]) < REL
        for l, kv in enumerate(o.kv):
            assert _rel(kv.keys, c["k"][i][l]) < REL
            assert _rel(kv.values, c["v"][i][l]) < REL
            assert kv.noise_tag == float(c["levels"][i]) and kv.conditioning_id == cond.id


def test_toy_runs_match_reference(golden, tiny_config, default_config):
    import paper_2511_20426_b200 as bc
    assert _rel(_stack(bc.run_cascade(tiny_config, "a red cube")), golden["tiny_cascade_bidir"]) < REL
    assert _rel(_stack(bc.run_cascade(bc.with_fields(tiny_config, attention_mode="causal"),
                                      "a red cube")), golden["tiny_cascade_causal"]) < REL
    seq = bc.run_sequential_reference(tiny_config, "a red cube")
    assert _rel(_stack(seq), golden["tiny_sequential"]) < REL
    d = default_config
    assert _rel(_stack(bc.run_cascade(d, "a red cube")), golden["default_cascade_bidir"]) < REL
    sw = [bc.SwitchSpec("a calm meadow after the storm", "cascade", at_block=8)]
    assert _rel(_stack(bc.run_cascade(d, "a lighthouse in a storm", switches=sw)),
                golden["default_cascade_switch8"]) < REL


@pytest.mark.parametrize("o", [2, 3, 4])
def test_toy_runs_every_offset_match_reference(golden, tiny_config, default_config, o):
    """Device runs at offsets 2..4 (batch widths 3/2/2 -- their own graph
    executables and attention work lists) vs the reference's outputs."""
    import paper_2511_20426_b200 as bc
    d = default_config
    assert _rel(_stack(bc.run_cascade(bc.with_fields(d, offset=o), "a red cube")),
                golden[f"default_cascade_o{o}"]) < REL
    assert _rel(_stack(bc.run_cascade(bc.with_fields(d, offset=o, attention_mode="causal"), "a red cube")),
                golden[f"default_causal_o{o}"]) < REL
    assert _rel(_stack(bc.run_cascade(bc.with_fields(tiny_config, offset=o), "a red cube")),
                golden[f"tiny_cascade_o{o}"]) < REL


def test_toy_recache_baseline_matches_reference(golden, default_config):
    """KV-recache comparison baseline on the device (fp64) vs the
    reference's own outputs, plus the sink refresh."""
    import paper_2511_20426_b200 as bc
    d = default_config
    rc = [bc.SwitchSpec("a calm meadow after the storm", "recache", at_block=8)]
    run = bc.run_cascade(d, "a lighthouse in a storm", switches=rc)
    assert _rel(_stack(run), golden["default_cascade_recache8"]) < REL
    assert run.switch_events[0].extra_passes == 7
    hit = next(e for e in run.trace.events if e.switch is not None)
    assert hit.wall_clock > 0 and 0 < hit.wall_seconds < hit.wall_clock
    rc5 = [bc.SwitchSpec("a calm meadow", "recache", at_block=5)]
    assert _rel(_stack(bc.run_cascade(bc.with_fields(d, attention_mode="causal"), "a red cube",
                                      switches=rc5)), golden["default_causal_recache5"]) < REL
    sw = [bc.SwitchSpec("a calm meadow after the storm", "cascade", at_block=8)]
    assert _rel(_stack(bc.run_cascade(bc.with_fields(d, refresh_sink_on_switch=True),
                                      "a lighthouse in a storm", switches=sw)),
                golden["default_refresh_sink8"]) < REL


def test_toy_recache_fixture_stream(default_config):
    """The reference's golden event stream (recache_session.jsonl) from the
    device engine: every non-pixel field identical, float32 pixels of all 13
    blocks within 1e-6 relative (fp64 device vs fp64 BLAS order)."""
    import base64
    import json
    import os
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200.stream import events_from_trace
    cfg = bc.with_fields(default_config, workers=5)
    run = bc.run_cascade(cfg, "a lighthouse in a storm",
                         switches=[bc.SwitchSpec("a calm meadow after the storm", "recache",
                                                 at_block=8)])
    with open(os.path.join(os.path.dirname(__file__), "golden", "recache_session.jsonl")) as fh:
        want = [json.loads(l) for l in fh if l.strip()]
    got = [json.loads(l) for l in events_from_trace(run.trace, cfg, run.outputs)]
    assert len(got) == len(want)

    def px(doc):
        return np.frombuffer(base64.b64decode(doc.pop("pixels")["data"]), dtype="<f4")
    for g, w in zip(got, want):
        if w["type"] == "block":
            a, b = px(g), px(w)
            assert _rel(a, b) < 1e-6
        assert g == w


def test_p1_equivalence_exact(default_config):
    """offset = passes reproduces the sequential rollout bit-for-bit
    (test_acceptance.py:27-40) -- on the device too."""
    import paper_2511_20426_b200 as bc
    ref = bc.run_sequential_reference(default_config, "a lighthouse in a storm")
    cas = bc.run_cascade(bc.with_fields(default_config, offset=5), "a lighthouse in a storm")
    assert np.array_equal(_stack(ref), _stack(cas))
    assert ref.emitted_order == cas.emitted_order


def test_worker_independence_exact(default_config):
    import paper_2511_20426_b200 as bc
    base = bc.run_cascade(default_config, "determinism")
    for g in (2, 5):
        other = bc.run_cascade(bc.with_fields(default_config, workers=g), "determinism")
        assert np.array_equal(_stack(base), _stack(other))
        assert base.pool.state_dump() == other.pool.state_dump()


def test_causal_truncation_invariance(default_config):
    import paper_2511_20426_b200 as bc
    for seed in range(5):
        cfg = bc.with_fields(default_config, attention_mode="causal", total_frames=18)
        full = bc.run_cascade(cfg, "p", session_seed=seed)
        trunc = bc.run_cascade(bc.with_fields(cfg, total_frames=12), "p", session_seed=seed)
        for b in range(4):
            assert np.array_equal(full.outputs[b], trunc.outputs[b])


def test_nonfinite_raises_iteration_error(default_config):
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200.scheduler import BatchPlan, PlanEntry
    w = bc.init_model(11, 2, 2, 16, 16)
    cond = bc.embed_prompt("executor prompt", 16)
    rng = np.random.default_rng(0)
    ents = [bc.EntryInput(0, rng.standard_normal((3, 16)), 1000.0, cond),
            bc.EntryInput(1, np.full((3, 16), np.nan), 1000.0, cond)]
    plan = BatchPlan(0, tuple(PlanEntry(b, 0, 1000.0, b % 2) for b in (0, 1)))
    mask = bc.build_mask([0, 1], [], "bidirectional", 3)
    with pytest.raises(bc.IterationError) as err:
        bc.execute(plan, ents, [], mask, w, bc.WorkerPool(2), bc.CostModel(), "bidirectional")
    assert err.value.block_index == 1


def test_wall_clock_trace(tiny_config):
    import paper_2511_20426_b200 as bc
    run = bc.run_cascade(tiny_config, "a red cube")
    walls = [e.wall_clock for e in run.trace.events]
    assert all(w > 0 for w in walls) and walls == sorted(walls)
    assert bc.instantaneous_fps(run.trace, clock="wall")[0].fps > 0
