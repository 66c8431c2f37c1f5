"""Print the measured Wan parity margins (rel-L2 vs the fp32 oracle) for
the committed tolerance table in DESIGN.md / profiles."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_20426_b200 as bc
from paper_2511_20426_b200 import engine
from paper_2511_20426_b200.wan import WanWeights, text_states
from oracle import wan as wo
from oracle.loop import wan_oracle_runtime
from oracle.schedule import visible_blocks


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / np.linalg.norm(b))


out = {}
for preset, over in (("tiny", {}), ("1.3b", {"layers": 2}), ("14b", {"layers": 1, "latent_height": 16,
                                                                    "latent_width": 16, "text_len": 128})):
    cfg = bc.wan_config(preset, total_frames=9, **over)
    w = WanWeights.random(cfg, 11)
    cond = bc.embed_prompt("a lighthouse in a storm", cfg.cond_dim)
    rng = np.random.default_rng(2)
    lat0 = rng.standard_normal((cfg.block_size, cfg.latent_dim)).astype(np.float32)
    pool = [bc.forward(w, [bc.EntryInput(0, lat0, 0.0, cond)], [], bc.build_mask([0], [], "causal", 3))[0].kv]
    batch, levels = [1, 2], [500.0, 1000.0]
    lat = {b: rng.standard_normal((cfg.block_size, cfg.latent_dim)).astype(np.float32) for b in batch}
    outs = bc.forward(w, [bc.EntryInput(b, lat[b], lv, cond) for b, lv in zip(batch, levels)], pool,
                      bc.build_mask(batch, [0], "bidirectional", 3))
    d = cfg.model_dim
    ref = wo.WanOracle(w.host_params(), cfg).forward(
        [(b, lat[b], lv) for b, lv in zip(batch, levels)],
        {0: [(l.keys.reshape(-1, d), l.values.reshape(-1, d)) for l in pool[0]]},
        visible_blocks(batch, [0], "bidirectional"), text_states(cond, cfg.text_len, cfg.text_dim))
    out[f"step_{preset}"] = [rel(o.x0, r[0].reshape(o.x0.shape)) for o, r in zip(outs, ref)]
cfg = bc.wan_config("tiny", total_frames=15)
w = WanWeights.random(cfg, 7)
params = w.host_params()
for mode, off in (("bidirectional", 1), ("causal", 1), ("bidirectional", 5)):
    c = bc.with_fields(cfg, attention_mode=mode, offset=off)
    g = bc.run_cascade(c, "a red cube", weights=w)
    orig = engine._runtime_for
    engine._runtime_for = wan_oracle_runtime(params)
    try:
        r = bc.run_cascade(c, "a red cube", weights=w)
    finally:
        engine._runtime_for = orig
    out[f"run_{mode}_o{off}"] = [rel(g.outputs[b], r.outputs[b]) for b in range(c.num_blocks)]
print(json.dumps(out, indent=1))
