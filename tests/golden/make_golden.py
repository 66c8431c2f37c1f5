"""Generate the golden vectors under tests/golden/ from the REFERENCE itself.

Run in the builder container (the reference is only there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src
(read-only) and records its outputs; nothing here is used at test time
except the files it writes.  The frontend fixture
pkg/frontend/test/fixtures/recache_session.jsonl (the reference's own golden
stream) is copied verbatim as recache_session.jsonl.
"""

from __future__ import annotations

import json
import os
import random
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import blockcascade as bc  # noqa: E402  (the reference)
from blockcascade.kvpool import KVPool  # noqa: E402

TINY = dict(layers=4, latent_dim=256, heads=2, head_dim=128, cond_dim=256,
            total_frames=18, offset=1, window_blocks=7, sink_blocks=1,
            attention_mode="bidirectional", pass_cost_base=1.0)


def run_outputs(cfg, prompt, **kw):
    return np.stack([v for _, v in sorted(bc.run_cascade(cfg, prompt, **kw).outputs.items())])


def seq_outputs(cfg, prompt, **kw):
    return np.stack([v for _, v in sorted(bc.run_sequential_reference(cfg, prompt, **kw).outputs.items())])


def forward_case(weights, batch_blocks, pool_blocks, levels, mode, seed, S=3):
    rng = np.random.default_rng(seed)
    d = weights.latent_dim
    cond = bc.embed_prompt(f"golden prompt {seed}", weights.cond_dim)
    pool = []
    for b in pool_blocks:
        m = bc.build_mask([b], [], "bidirectional", S)
        e = bc.EntryInput(b, rng.standard_normal((S, d)), 0.0, cond)
        pool.append(bc.forward(weights, [e], [], m)[0].kv)
    ents = [bc.EntryInput(b, rng.standard_normal((S, d)), lv, cond)
            for b, lv in zip(batch_blocks, levels)]
    mask = bc.build_mask(batch_blocks, pool_blocks, mode, S)
    outs = bc.forward(weights, ents, pool, mask)
    case = {
        "batch": np.array(batch_blocks), "pool": np.array(pool_blocks),
        "levels": np.array(levels, dtype=np.float64), "mode": np.array(mode),
        "prompt": np.array(f"golden prompt {seed}"),
        "latents": np.stack([e.latents for e in ents]),
        "pool_k": np.stack([np.stack([kv.keys for kv in p]) for p in pool]) if pool else np.zeros(0),
        "pool_v": np.stack([np.stack([kv.values for kv in p]) for p in pool]) if pool else np.zeros(0),
        "x0": np.stack([o.x0 for o in outs]),
        "k": np.stack([np.stack([kv.keys for kv in o.kv]) for o in outs]),
        "v": np.stack([np.stack([kv.values for kv in o.kv]) for o in outs]),
    }
    return case


def main():
    arrays = {}
    # ---- full runs (config 1 tiny, default toy config) ----
    tiny = bc.CascadeConfig(**TINY).validate()
    arrays["tiny_cascade_bidir"] = run_outputs(tiny, "a red cube")
    arrays["tiny_cascade_causal"] = run_outputs(bc.with_fields(tiny, attention_mode="causal"), "a red cube")
    arrays["tiny_sequential"] = seq_outputs(tiny, "a red cube")
    dflt = bc.CascadeConfig(total_frames=39, pass_cost_base=1.0).validate()
    arrays["default_cascade_bidir"] = run_outputs(dflt, "a red cube")
    arrays["default_cascade_causal"] = run_outputs(bc.with_fields(dflt, attention_mode="causal"), "a red cube")
    arrays["default_sequential"] = seq_outputs(dflt, "a red cube")
    arrays["default_cascade_o2"] = run_outputs(bc.with_fields(dflt, offset=2), "a red cube")
    # every offset the reference sweeps (test_acceptance.py:42-55): batch widths 3/2/2
    for o in (2, 3, 4):
        if o != 2:
            arrays[f"default_cascade_o{o}"] = run_outputs(bc.with_fields(dflt, offset=o), "a red cube")
        arrays[f"default_causal_o{o}"] = run_outputs(bc.with_fields(dflt, offset=o, attention_mode="causal"),
                                                     "a red cube")
        arrays[f"tiny_cascade_o{o}"] = run_outputs(bc.with_fields(tiny, offset=o), "a red cube")
    sw = [bc.SwitchSpec("a calm meadow after the storm", "cascade", at_block=8)]
    arrays["default_cascade_switch8"] = run_outputs(dflt, "a lighthouse in a storm", switches=sw)
    # KV-recache comparison baseline and the sink refresh (both rebuild pool KV)
    rc = [bc.SwitchSpec("a calm meadow after the storm", "recache", at_block=8)]
    arrays["default_cascade_recache8"] = run_outputs(dflt, "a lighthouse in a storm", switches=rc)
    rc5 = [bc.SwitchSpec("a calm meadow", "recache", at_block=5)]
    arrays["default_causal_recache5"] = run_outputs(bc.with_fields(dflt, attention_mode="causal"),
                                                    "a red cube", switches=rc5)
    arrays["default_refresh_sink8"] = run_outputs(bc.with_fields(dflt, refresh_sink_on_switch=True),
                                                  "a lighthouse in a storm", switches=sw)
    # ---- operator cases: forward with pool + batch ----
    w_small = bc.init_model(11, 2, 2, 16, 16)
    w_tiny = bc.init_model(7, 4, 2, 256, 256)
    cases = {
        "small_bidir": forward_case(w_small, [1, 2], [0], [750.0, 1000.0], "bidirectional", 1),
        "small_causal": forward_case(w_small, [4, 5, 6], [0, 2, 3], [250.0, 500.0, 1000.0], "causal", 2),
        "tiny_bidir5": forward_case(w_tiny, [3, 4, 5, 6, 7], [0, 1, 2],
                                    [0.0, 250.0, 500.0, 750.0, 1000.0], "bidirectional", 3),
        "tiny_causal5": forward_case(w_tiny, [3, 4, 5, 6, 7], [0, 1, 2],
                                     [0.0, 250.0, 500.0, 750.0, 1000.0], "causal", 4),
        "tiny_single": forward_case(w_tiny, [0], [], [1000.0], "bidirectional", 5),
    }
    for name, case in cases.items():
        for k, v in case.items():
            arrays[f"case_{name}_{k}"] = v
    # ---- noise / prompt KATs ----
    ns = bc.NoiseStream(20260809, 16)
    keys = [(0, 0, 0), (1, 2, 3), (12, 4, 38), (79, 3, 239)]
    arrays["noise_keys"] = np.array(keys)
    arrays["noise_draws"] = np.stack([ns.draw(*k) for k in keys])
    arrays["noise_wan_block"] = bc.NoiseStream(20260809, 99840).block_noise(5, 2, 15, 3)[:, :4096]
    prompts = ["a red cube", "a lighthouse in a storm", "Ω unicode ✔"]
    arrays["prompt_embed"] = np.stack([bc.embed_prompt(p, 256).embedding for p in prompts])
    arrays["prompt_ids"] = np.array([bc.embed_prompt(p, 16).id for p in prompts])
    arrays["renoise_x0"] = np.random.default_rng(0).standard_normal((3, 16))
    arrays["renoise_eps"] = np.random.default_rng(1).standard_normal((3, 16))
    arrays["renoise_750"] = bc.renoise(arrays["renoise_x0"], arrays["renoise_eps"], 750.0)
    arrays["renoise_333"] = bc.renoise(arrays["renoise_x0"], arrays["renoise_eps"], 333.0)
    np.savez_compressed(os.path.join(HERE, "toy_golden.npz"), **arrays)

    # ---- schedules, pools, masks (JSON) ----
    sched = bc.make_schedule([1000, 750, 500, 250])
    plans = {}
    for o in range(1, 6):
        for blocks in (1, 2, 5, 6, 13, 20, 80):
            st = bc.CascadeState(num_blocks=blocks, offset=o, schedule=sched, workers=5)
            rows = []
            while not st.done:
                p = bc.plan_iteration(st)
                rows.append([[e.block_index, e.pass_index, e.noise_level, e.worker] for e in p.entries])
                bc.advance(st, p, p.blocks)
            plans[f"{blocks}_{o}"] = rows
    rng = random.Random(20260809)
    pools = []
    for _ in range(300):
        window, sink = rng.randint(1, 8), rng.choice([0, 1])
        inserts = [rng.randint(0, 30) for _ in range(rng.randint(0, 25))]
        if sink and rng.random() < 0.8:
            inserts.insert(0, 0)
        pool = KVPool.empty(window, sink)
        trail = []
        for b in inserts:
            pool = pool.insert(b, (bc.LayerKV(b, 0, np.zeros((1, 1, 1)), np.zeros((1, 1, 1)), 0.0, "x"),))
            trail.append(list(pool.block_indices))
        pools.append({"window": window, "sink": sink, "inserts": inserts, "trail": trail})
    masks = []
    for _ in range(300):
        blocks = rng.sample(range(24), k=rng.randint(1, 7))
        batch = sorted(blocks[: rng.randint(1, len(blocks))])
        pool = sorted(set(blocks) - set(batch))
        mode = rng.choice(["causal", "bidirectional"])
        size = rng.choice([1, 2, 3])
        m = bc.build_mask(batch, pool, mode, size)
        masks.append({"batch": batch, "pool": pool, "mode": mode, "size": size,
                      "visible": [m.visible_key_blocks(b) for b in m.batch_blocks],
                      "matrix_sum": int(m.matrix.sum()), "shape": list(m.matrix.shape)})
    tiny_run = bc.run_cascade(tiny, "a red cube")
    trace = [json.loads(e.to_json()) for e in tiny_run.trace.events]
    for ev in trace:
        ev.pop("wall_seconds"), ev.pop("wall_clock")
    with open(os.path.join(HERE, "schedule_golden.json"), "w") as fh:
        json.dump({"plans": plans, "pools": pools, "masks": masks, "tiny_trace": trace}, fh)
    shutil.copyfile("/root/reference/pkg/frontend/test/fixtures/recache_session.jsonl",
                    os.path.join(HERE, "recache_session.jsonl"))
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
