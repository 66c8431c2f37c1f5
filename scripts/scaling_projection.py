"""Projected multi-GPU scaling from ONE GPU (a projection, not a
measurement): the emulated ranks run each rank's kernels alone on the whole
GPU (stage-interleaved on one stream), so a rank's summed kernel time per
iteration is the compute time one GPU of a G-GPU job would spend; the
iteration time is the max over ranks.  NVLink transfer time is NOT included
(the P2P K/V stores go to the same device here), nor is host noise.
Prints projected generated frames/s of the 13-block Wan-1.3B cascade for
both partitions and G = 1, 2, 4, 5, 8."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["BC_EMULATE_TIMING"] = "1"
import paper_2511_20426_b200 as bc
from paper_2511_20426_b200 import distributed
from paper_2511_20426_b200.wan import ResidentNoiseFeed, WanWeights, run_noise_keys

cfg = bc.wan_config(os.environ.get("PRESET", "1.3b"), total_frames=39)
w = WanWeights.random(cfg, 7)
feed = ResidentNoiseFeed(20260809, cfg, run_noise_keys(cfg))
frames = cfg.num_blocks * 12
res = {}
distributed.EMULATE = True
captured = {}
orig_close = distributed.EmulatedRanks.close


def close(self):
    captured["t"] = self.rank_times
    orig_close(self)


distributed.EmulatedRanks.close = close
for shard in ("rows", "blocks"):
    os.environ["BC_TEMPORAL_SHARD"] = shard
    for g in (2, 4, 5, 8):
        conf = bc.with_fields(cfg, workers=g)
        bc.run_cascade(conf, "p", weights=w, noise_feed=feed)   # warm-up
        run = bc.run_cascade(conf, "p", weights=w, noise_feed=feed)
        t = captured["t"]
        it_ms = [max(r) for r in t]
        busy = [sum(r[k] for r in t) for k in range(g)]
        fps = frames / (sum(it_ms) / 1e3)
        res[f"{shard}_G{g}"] = {"projected_fps": round(fps, 1), "iteration_ms_sum": round(sum(it_ms), 1),
                                "rank_busy_ms": [round(x, 1) for x in busy]}
        print(shard, g, res[f"{shard}_G{g}"], flush=True)
distributed.EMULATE = False
run = bc.run_cascade(cfg, "p", weights=w, noise_feed=feed)
run = bc.run_cascade(cfg, "p", weights=w, noise_feed=feed)
one = sum(e.wall_seconds for e in run.trace.events)
res["G1_measured"] = {"fps": round(frames / one, 1), "iteration_ms_sum": round(one * 1e3, 1)}
print(json.dumps(res))
