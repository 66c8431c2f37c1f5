"""Emulated multi-rank (one process, G rank contexts stage-interleaved on one
stream) at full Wan-1.3B token geometry with few layers: rows and blocks
partitions vs the single-rank run, bit-identical outputs required."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_20426_b200 as bc
from paper_2511_20426_b200 import distributed
from paper_2511_20426_b200.wan import WanWeights

cfg = bc.wan_config("1.3b", total_frames=3 * int(os.environ.get("BLOCKS", "7")),
                    layers=int(os.environ.get("LAYERS", "2")))
w = WanWeights.random(cfg, 7)
base = bc.run_cascade(cfg, "full", weights=w)
distributed.EMULATE = True
for shard in ("rows", "blocks"):
    os.environ["BC_TEMPORAL_SHARD"] = shard
    for g in (2, 3, 8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run = bc.run_cascade(bc.with_fields(cfg, workers=g), "full", weights=w)
        torch.cuda.synchronize()
        same = all(np.array_equal(run.outputs[b], base.outputs[b]) for b in base.outputs)
        print(f"{shard} G={g}: {time.perf_counter() - t0:.2f} s, bit-identical {same}", flush=True)
