"""Host profile of the device toy path (reference config 1) -- where do the
~17 ms per run go?"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_20426_b200 as bc

cfg = bc.CascadeConfig(layers=4, latent_dim=256, heads=2, head_dim=128, cond_dim=256, total_frames=18,
                       offset=1, window_blocks=7, sink_blocks=1, attention_mode="bidirectional").validate()
w = bc.init_model(7, 4, 2, 256, 256)
for _ in range(3):
    bc.run_cascade(cfg, "a red cube", weights=w)
torch.cuda.synchronize()
t = time.perf_counter()
bc.run_cascade(cfg, "a red cube", weights=w)
torch.cuda.synchronize()
print("ms per run", (time.perf_counter() - t) * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    bc.run_cascade(cfg, "a red cube", weights=w)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
