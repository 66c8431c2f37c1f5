"""Run one Wan-1.3B cascade generation and open the CUDA profiler range
around ONE steady-state iteration (width 5, 13 visible blocks), for ncu:

  ncu --profile-from-start off ... python scripts/profile_iter.py [--iteration 9]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_20426_b200 as bc  # noqa: E402
from paper_2511_20426_b200 import wan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iteration", type=int, default=9)
ap.add_argument("--preset", default="1.3b")
ap.add_argument("--layers", type=int, default=0)
args = ap.parse_args()
over = {"layers": args.layers} if args.layers else {}
cfg = bc.wan_config(args.preset, total_frames=39, **over)
w = wan.WanWeights.random(cfg, 7)
feed = wan.ResidentNoiseFeed(20260809, cfg, wan.run_noise_keys(cfg))
orig = wan.WanSession.step


def step(self, plan, *a, **k):
    hit = plan.iteration == args.iteration
    if hit:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
    orig(self, plan, *a, **k)
    if hit:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()


wan.WanSession.step = step
bc.run_cascade(cfg, "a lighthouse in a storm", weights=w, noise_feed=feed)
print("profiled iteration", args.iteration)
