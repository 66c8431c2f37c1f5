"""Per-kernel-class GPU time of one 13-block Wan-1.3B cascade generation in
the PRODUCT launch mode (CUDA graphs, no per-kernel events), from CUPTI
activity records via torch.profiler -- beside the bench's eager,
event-bracketed class breakdown.  Prints JSON: class -> (ms, launches)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2511_20426_b200 as bc  # noqa: E402
from paper_2511_20426_b200.wan import ResidentNoiseFeed, WanWeights, run_noise_keys  # noqa: E402


def classify(names):
    """attention launches alternate self / cross within a layer (same kernel)."""
    out, attn_k = [], 0
    for n in names:
        if "attn_sched_kernel" in n or "attn_kernel" in n:
            out.append("self_attention" if attn_k % 2 == 0 else "cross_attention")
            attn_k += 1
        elif "gemm_kernel" in n:
            out.append("gemm")
        else:
            out.append("bandwidth")
    return out


def main():
    cfg = bc.wan_config(os.environ.get("PRESET", "1.3b"), total_frames=39)
    w = WanWeights.random(cfg, 7)
    feed = ResidentNoiseFeed(20260809, cfg, run_noise_keys(cfg))
    for _ in range(2):
        bc.run_cascade(cfg, "p", weights=w, noise_feed=feed)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        bc.run_cascade(cfg, "p", weights=w, noise_feed=feed)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
           and "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
    evs.sort(key=lambda e: e.time_range.start)
    mine = [e for e in evs if "bc::" in e.name or "gemm_kernel" in e.name or "_kernel" in e.name]
    res = {}
    for e, c in zip(mine, classify([e.name for e in mine])):
        ms, n = res.get(c, (0.0, 0))
        res[c] = (ms + (e.time_range.end - e.time_range.start) / 1e3, n + 1)
    span = (mine[-1].time_range.end - mine[0].time_range.start) / 1e3 if mine else 0.0
    print(json.dumps({"classes": {k: {"ms": round(v[0], 3), "launches": v[1]} for k, v in res.items()},
                      "kernels": len(mine), "span_ms": round(span, 1),
                      "names": sorted({e.name[:80] for e in mine})[:40]}))


if __name__ == "__main__":
    main()
