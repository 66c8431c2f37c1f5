"""Multi-rank smoke run under torchrun (any backend; BC_FORCE_DEVICE lets
several ranks share one GPU for testing): one Wan-shaped cascade per
configuration with per-run wall time, outputs compared with a one-process
run on rank 0.  usage:
  BC_FORCE_DEVICE=0 torchrun --nproc-per-node 2 scripts/dist_smoke.py [--preset 1.3b --layers 2]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="tiny")
ap.add_argument("--layers", type=int, default=0)
ap.add_argument("--blocks", type=int, default=6)
args = ap.parse_args()
rank, local = int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(int(os.environ.get("BC_FORCE_DEVICE", local)))
dist.init_process_group(os.environ.get("BC_DIST_BACKEND", "gloo"))
import paper_2511_20426_b200 as bc
from paper_2511_20426_b200.wan import WanWeights
over = {"layers": args.layers} if args.layers else {}
cfg = bc.wan_config(args.preset, total_frames=3 * args.blocks, **over)
w = WanWeights.random(cfg, 7)
for i in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run = bc.run_cascade(cfg, "smoke", weights=w)
    torch.cuda.synchronize()
    print(f"rank {rank} run {i}: {time.perf_counter() - t0:.2f} s, {run.iterations} iterations", flush=True)
outs = {b: run.outputs[b] for b in run.outputs}
dist.barrier()
dist.destroy_process_group()
if rank == 0:
    ref = bc.run_cascade(cfg, "smoke", weights=w)   # single-process session (no group)
    same = all(np.array_equal(outs[b], ref.outputs[b]) for b in ref.outputs)
    print(f"rank 0: multi-rank outputs bit-identical to the single-process run: {same}", flush=True)
