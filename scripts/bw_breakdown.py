"""Per-kernel breakdown of one 13-block Wan-1.3B cascade (SEQ=1: the
sequential rollout) in the product launch
mode (CUDA graphs, no per-kernel events): CUPTI durations (torch.profiler)
summed by kernel name, with the launch count and the mean / min / max
duration -- where the bandwidth class's time goes."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2511_20426_b200 as bc
from paper_2511_20426_b200.wan import ResidentNoiseFeed, WanWeights, run_noise_keys

cfg = bc.wan_config(os.environ.get("PRESET", "1.3b"), total_frames=39)
if os.environ.get("SEQ"):  # the sequential (width-1) rollout instead of the cascade
    cfg = bc.with_fields(cfg, offset=cfg.passes)
w = WanWeights.random(cfg, 7)
feed = ResidentNoiseFeed(20260809, cfg, run_noise_keys(cfg))
for _ in range(2):
    bc.run_cascade(cfg, "p", weights=w, noise_feed=feed)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as p:
    bc.run_cascade(cfg, "p", weights=w, noise_feed=feed)
    torch.cuda.synchronize()
agg = defaultdict(list)
for e in p.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:60]].append((e.time_range.end - e.time_range.start) / 1e3)
tot = sum(sum(v) for v in agg.values())
print(f"total kernel time {tot:.1f} ms")
for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):9.2f} ms {100 * sum(v) / tot:5.1f}%  n={len(v):5d}  mean {1e3 * sum(v) / len(v):8.1f} us"
          f"  min {1e3 * min(v):8.1f}  max {1e3 * max(v):8.1f}  {name}")
if os.environ.get("LIST"):  # per-launch durations of one kernel, in launch order (first 12)
    evs = sorted((e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA
                  and os.environ["LIST"] in e.name), key=lambda e: e.time_range.start)
    print(os.environ["LIST"], [round(e.time_range.end - e.time_range.start, 1) for e in evs[:12]], "us")
