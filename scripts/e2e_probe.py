"""Where does the end-to-end (host-noise) run lose time against the
device-resident run?  Prints wall time, summed GPU iteration time and the
host-side gaps at start / end of a run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_20426_b200 as bc
from paper_2511_20426_b200.wan import ResidentNoiseFeed, WanWeights, run_noise_keys
cfg = bc.wan_config("1.3b", total_frames=39)
w = WanWeights.random(cfg, 7)
feed = ResidentNoiseFeed(20260809, cfg, run_noise_keys(cfg))
for label, nf in (("resident", feed), ("host", None), ("resident", feed), ("host", None)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = bc.run_cascade(cfg, "a red cube", session_seed=20260809, weights=w, noise_feed=nf)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    gpu = sum(e.wall_seconds for e in r.trace.events)
    print(f"{label:9s} wall {wall*1e3:7.1f} ms  gpu-iterations {gpu*1e3:7.1f} ms  last wall_clock {r.trace.events[-1].wall_clock*1e3:7.1f}")

# host-side cost of opening / closing a session (inside every run_cascade)
from paper_2511_20426_b200 import wan
orig_init, orig_close = wan.WanSession.__init__, wan.WanSession.close
acc = {"open": 0.0, "close": 0.0}


def init(self, *a, **k):
    torch.cuda.synchronize()
    t = time.perf_counter()
    orig_init(self, *a, **k)
    torch.cuda.synchronize()
    acc["open"] += time.perf_counter() - t


def close(self):
    t = time.perf_counter()
    orig_close(self)
    acc["close"] += time.perf_counter() - t


wan.WanSession.__init__, wan.WanSession.close = init, close
for label, nf in (("resident", feed), ("host", None)):
    acc.update(open=0.0, close=0.0)
    t0 = time.perf_counter()
    r = bc.run_cascade(cfg, "a red cube", session_seed=20260809, weights=w, noise_feed=nf)
    torch.cuda.synchronize()
    print(f"{label:9s} wall {(time.perf_counter() - t0)*1e3:7.1f} ms  session open {acc['open']*1e3:6.1f} ms  close {acc['close']*1e3:6.1f} ms")
