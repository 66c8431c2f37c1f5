"""Pin the CPU oracle (and the product's host logic) to vectors the reference
itself produced (tests/golden/make_golden.py).  CPU only."""

import base64
import json
import os

import numpy as np
import pytest

from oracle import schedule as sched_oracle
from oracle import toy as toy_oracle

CASES = ["small_bidir", "small_causal", "tiny_bidir5", "tiny_causal5", "tiny_single"]


def _weights_for(name):
    from paper_2511_20426_b200 import init_model
    if name.startswith("small"):
        return init_model(11, 2, 2, 16, 16)
    return init_model(7, 4, 2, 256, 256)


def _case(golden, name):
    return {k[len(f"case_{name}_"):]: v for k, v in golden.items() if k.startswith(f"case_{name}_")}


@pytest.mark.parametrize("name", CASES)
def test_toy_oracle_forward_bit_exact(golden, name):
    from paper_2511_20426_b200 import embed_prompt
    c = _case(golden, name)
    w = toy_oracle.weights_from(_weights_for(name))
    cond = embed_prompt(str(c["prompt"]), w["w_cond"].shape[1])
    batch = [int(b) for b in c["batch"]]
    pool = [int(b) for b in c["pool"]]
    pool_kv = {b: [(c["pool_k"][i][l], c["pool_v"][i][l]) for l in range(c["pool_k"].shape[1])]
               for i, b in enumerate(pool)}
    vis = sched_oracle.visible_blocks(batch, pool, str(c["mode"]))
    ents = [(b, c["latents"][i], float(c["levels"][i]), cond.embedding) for i, b in enumerate(batch)]
    outs = toy_oracle.forward(w, ents, pool_kv, vis)
    for i, (x0, kv) in enumerate(outs):
        assert np.array_equal(x0, c["x0"][i])
        for l, (k, v) in enumerate(kv):
            assert np.array_equal(k, c["k"][i][l])
            assert np.array_equal(v, c["v"][i][l])


def test_toy_weights_identical_to_reference(golden):
    """init_model draws the reference's exact weights (needed for parity)."""
    from paper_2511_20426_b200 import init_model
    import sys
    sys.path.insert(0, "/root/reference/pkg/src") if os.path.isdir("/root/reference") else None
    w = init_model(7, 4, 2, 256, 256)
    c = _case(golden, "tiny_single")
    outs = toy_oracle.forward(toy_oracle.weights_from(w),
                              [(0, c["latents"][0], 1000.0,
                                __import__("paper_2511_20426_b200").embed_prompt(
                                    str(c["prompt"]), 256).embedding)], {}, {0: [0]})
    assert np.array_equal(outs[0][0], c["x0"][0])


def test_noise_and_prompt_kats(golden):
    from paper_2511_20426_b200 import NoiseStream, embed_prompt
    ns = NoiseStream(20260809, 16)
    for key, want in zip(golden["noise_keys"], golden["noise_draws"]):
        assert np.array_equal(ns.draw(*[int(x) for x in key]), want)
    wan = NoiseStream(20260809, 99840)
    assert np.array_equal(wan.block_noise(5, 2, 15, 3)[:, :4096], golden["noise_wan_block"])
    f32 = wan.block_noise_f32(5, 2, 15, 3)
    assert np.array_equal(f32[:, :4096], golden["noise_wan_block"].astype(np.float32))
    for p, emb, pid in zip(["a red cube", "a lighthouse in a storm", "Ω unicode ✔"],
                           golden["prompt_embed"], golden["prompt_ids"]):
        c = embed_prompt(p, 256)
        assert np.array_equal(c.embedding, emb)
        assert embed_prompt(p, 16).id == str(pid)


def test_renoise_oracle_bit_exact(golden):
    for lv in (750.0, 333.0):
        got = toy_oracle.renoise(golden["renoise_x0"], golden["renoise_eps"], lv)
        assert np.array_equal(got, golden[f"renoise_{int(lv)}"])


# ---------------------------------------------------------------------------
# host logic vs reference plans / pools / masks
# ---------------------------------------------------------------------------

def test_plans_match_reference(golden_sched):
    from paper_2511_20426_b200 import CascadeState, advance, make_schedule, plan_iteration
    from paper_2511_20426_b200.scheduler import timestep_table
    sched = make_schedule([1000, 750, 500, 250])
    for key, rows in golden_sched["plans"].items():
        blocks, o = (int(x) for x in key.split("_"))
        st = CascadeState(num_blocks=blocks, offset=o, schedule=sched, workers=5)
        got = []
        while not st.done:
            p = plan_iteration(st)
            got.append([[e.block_index, e.pass_index, e.noise_level, e.worker] for e in p.entries])
            advance(st, p, p.blocks)
        assert got == rows, key
        table = timestep_table(blocks, sched, o)
        assert [[[b, p, lv] for b, p, lv in it] for it in table] == \
               [[r[:3] for r in it] for it in rows]
        assert [[(b, p) for b, p, _ in it] for it in table] == \
               sched_oracle.enumerate_schedule(blocks, 5, o)


def test_pools_match_reference(golden_sched):
    from paper_2511_20426_b200 import KVPool, LayerKV
    for case in golden_sched["pools"]:
        pool = KVPool.empty(case["window"], case["sink"])
        for b, want in zip(case["inserts"], case["trail"]):
            pool = pool.insert(b, (LayerKV(b, 0, np.zeros((1, 1, 1)), np.zeros((1, 1, 1)), 0.0, "x"),))
            assert pool.block_indices == want
        assert pool.block_indices == sched_oracle.replay_pool(case["inserts"], case["window"],
                                                              case["sink"])[0]


def test_masks_match_reference(golden_sched):
    from paper_2511_20426_b200 import build_mask
    from paper_2511_20426_b200.denoiser import visible_block_lists
    for m in golden_sched["masks"]:
        mask = build_mask(m["batch"], m["pool"], m["mode"], m["size"])
        assert visible_block_lists(mask) == m["visible"]
        assert int(mask.matrix.sum()) == m["matrix_sum"]
        assert list(mask.matrix.shape) == m["shape"]
        vis = sched_oracle.visible_blocks(m["batch"], m["pool"], m["mode"])
        assert [vis[b] for b in mask.batch_blocks] == m["visible"]


# ---------------------------------------------------------------------------
# product engine (host logic) driven by the oracle forward == reference runs
# ---------------------------------------------------------------------------

def _stack(run):
    return np.stack([run.outputs[k] for k in sorted(run.outputs)])


@pytest.mark.parametrize("o", [2, 3, 4])
def test_engine_runs_every_offset_match_reference(oracle_engine, golden, tiny_config, default_config, o):
    """Offsets 2..4 (batch widths 3/2/2; reference test_acceptance.py:42-55)."""
    from paper_2511_20426_b200 import run_cascade, with_fields
    d = default_config
    assert np.array_equal(_stack(run_cascade(with_fields(d, offset=o), "a red cube")),
                          golden[f"default_cascade_o{o}"])
    assert np.array_equal(_stack(run_cascade(with_fields(d, offset=o, attention_mode="causal"), "a red cube")),
                          golden[f"default_causal_o{o}"])
    assert np.array_equal(_stack(run_cascade(with_fields(tiny_config, offset=o), "a red cube")),
                          golden[f"tiny_cascade_o{o}"])


def test_engine_runs_match_reference(oracle_engine, golden, tiny_config, default_config):
    from paper_2511_20426_b200 import SwitchSpec, run_cascade, run_sequential_reference, with_fields
    assert np.array_equal(_stack(run_cascade(tiny_config, "a red cube")), golden["tiny_cascade_bidir"])
    assert np.array_equal(_stack(run_cascade(with_fields(tiny_config, attention_mode="causal"),
                                             "a red cube")), golden["tiny_cascade_causal"])
    assert np.array_equal(_stack(run_sequential_reference(tiny_config, "a red cube")),
                          golden["tiny_sequential"])
    d = default_config
    assert np.array_equal(_stack(run_cascade(d, "a red cube")), golden["default_cascade_bidir"])
    assert np.array_equal(_stack(run_cascade(with_fields(d, attention_mode="causal"), "a red cube")),
                          golden["default_cascade_causal"])
    assert np.array_equal(_stack(run_cascade(with_fields(d, offset=2), "a red cube")),
                          golden["default_cascade_o2"])
    assert np.array_equal(_stack(run_sequential_reference(d, "a red cube")),
                          golden["default_sequential"])
    assert np.array_equal(_stack(run_cascade(with_fields(d, offset=5), "a red cube")),
                          golden["default_sequential"])
    sw = [SwitchSpec("a calm meadow after the storm", "cascade", at_block=8)]
    assert np.array_equal(_stack(run_cascade(d, "a lighthouse in a storm", switches=sw)),
                          golden["default_cascade_switch8"])


def test_recache_baseline_runs_match_reference(oracle_engine, golden, default_config):
    """KV-recache comparison baseline (reference kvpool.recache,
    engine._apply_switch) and the sink refresh, through the product engine."""
    from paper_2511_20426_b200 import SwitchSpec, run_cascade, with_fields
    d = default_config
    rc = [SwitchSpec("a calm meadow after the storm", "recache", at_block=8)]
    run = run_cascade(d, "a lighthouse in a storm", switches=rc)
    assert np.array_equal(_stack(run), golden["default_cascade_recache8"])
    ev = run.switch_events[0]
    assert (ev.extra_passes, ev.stall_modeled) == (7, 7.0)
    rc5 = [SwitchSpec("a calm meadow", "recache", at_block=5)]
    assert np.array_equal(_stack(run_cascade(with_fields(d, attention_mode="causal"), "a red cube",
                                             switches=rc5)), golden["default_causal_recache5"])
    sw = [SwitchSpec("a calm meadow after the storm", "cascade", at_block=8)]
    ref = run_cascade(with_fields(d, refresh_sink_on_switch=True), "a lighthouse in a storm",
                      switches=sw)
    assert np.array_equal(_stack(ref), golden["default_refresh_sink8"])
    assert ref.switch_events[0].extra_passes == 1


def test_engine_trace_matches_reference(oracle_engine, golden_sched, tiny_config):
    from paper_2511_20426_b200 import run_cascade
    run = run_cascade(tiny_config, "a red cube")
    got = [json.loads(e.to_json()) for e in run.trace.events]
    for ev in got:
        ev.pop("wall_seconds"), ev.pop("wall_clock")
    assert got == golden_sched["tiny_trace"]


def test_recache_fixture_full_stream(oracle_engine, default_config):
    """The reference's own golden stream (frontend fixture
    recache_session.jsonl: 13 blocks, G=5, a recache switch at block 8),
    reproduced byte for byte -- every switch/metrics/block/done line incl.
    the float32-decoded pixels -- by the product engine + event projection
    driven by the oracle forward."""
    from paper_2511_20426_b200 import SwitchSpec, run_cascade, with_fields
    from paper_2511_20426_b200.stream import events_from_trace
    cfg = with_fields(default_config, workers=5)
    run = run_cascade(cfg, "a lighthouse in a storm",
                      switches=[SwitchSpec("a calm meadow after the storm", "recache", at_block=8)])
    with open(os.path.join(os.path.dirname(__file__), "golden", "recache_session.jsonl")) as fh:
        want = [l.rstrip("\n") for l in fh if l.strip()]
    got = events_from_trace(run.trace, cfg, run.outputs)
    assert len(got) == len(want) == 32
    for g, w in zip(got, want):
        assert g == w
