"""Per-iteration device time of one 13-block Wan-1.3B cascade (and the
sequential rollout): width, visible blocks, algorithmic TFLOP and achieved
TFLOP/s per iteration -- where fill / drain iterations lose efficiency."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_20426_b200 as bc
from paper_2511_20426_b200.wan import ResidentNoiseFeed, WanWeights, run_noise_keys

cfg = bc.wan_config(os.environ.get("PRESET", "1.3b"), total_frames=39)
w = WanWeights.random(cfg, 7)
feed = ResidentNoiseFeed(20260809, cfg, run_noise_keys(cfg))
d, L, T, ffn, tl = cfg.model_dim, cfg.layers, cfg.tokens_per_block, cfg.ffn_dim, cfg.text_len


def flops(entries):
    tot = 0.0
    for e in entries:
        nk = e["visible_frames"] // cfg.block_size * T
        tot += L * (2 * T * d * 3 * d + 3 * 2 * T * d * d + 4 * T * d * ffn + 4 * T * nk * d + 4 * T * tl * d)
    return tot


for kind, conf in (("cascade", cfg), ("sequential", bc.with_fields(cfg, offset=cfg.passes))):
    for _ in range(2):
        run = bc.run_cascade(conf, "p", weights=w, noise_feed=feed)
    tot_t = tot_f = 0.0
    for ev in run.trace.events:
        f = flops(ev.entries)
        tot_t += ev.wall_seconds
        tot_f += f
        if kind == "cascade":
            print(f"{kind} it {ev.iteration:2d} width {len(ev.entries)} vis {[e['visible_frames'] // 3 for e in ev.entries]} "
                  f"{ev.wall_seconds * 1e3:7.1f} ms  {f / 1e12:6.1f} TF  {f / ev.wall_seconds / 1e12:6.0f} TFLOP/s")
    print(f"{kind}: {tot_t * 1e3:.0f} ms, {tot_f / 1e15:.3f} PF, {tot_f / tot_t / 1e12:.0f} TFLOP/s overall")
