"""Time the streaming VAE decode of Wan2.1-geometry blocks (3 latent frames
-> 12 video frames at 480x832) on cuda:0: ms per block, algorithmic
TFLOP/s, and the per-kernel split with BC_VAE_PROFILE=1 (torch profiler
free: CUDA events around each decoder op class)."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights, vae_config  # noqa: E402


def main():
    cfg = vae_config("wan2.1")
    dec = VaeDecoder(VaeWeights.random(cfg, 11))
    dec.reset()
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    zs = [torch.randn((3, 16, cfg.latent_h, cfg.latent_w), generator=g, device="cuda") for _ in range(6)]
    dec.decode_block(zs[0])
    dec.decode_block(zs[1])
    torch.cuda.synchronize()
    times = []
    for z in zs[2:]:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dec.stream)
        dec.decode_block(z)
        e1.record(dec.stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    dec.profile(True)
    dec.decode_block(zs[2])
    prof = dec.profile_report()
    ms = sorted(times)[len(times) // 2]
    fl = dec.flops_per_block(False)
    print(json.dumps({"ms_per_block": ms, "ms_all": times, "tflop_per_block": fl / 1e12,
                      "tflops": fl / ms / 1e9, "video_frames_per_block": 12,
                      "decode_fps": 12 / ms * 1e3, "buffers_gb": dec.nbytes() / 1e9,
                      "profile": dict(sorted(prof.items(), key=lambda kv: -kv[1]["ms"]))}, indent=1))


if __name__ == "__main__":
    main()
