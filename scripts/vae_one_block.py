"""Decode a few Wan2.1-geometry blocks (ncu target: the launch list of one
steady-state block decode)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights, vae_config  # noqa: E402

cfg = vae_config("wan2.1")
dec = VaeDecoder(VaeWeights.random(cfg, 11))
dec.reset()
g = torch.Generator(device="cuda")
g.manual_seed(1)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    dec.decode_block(torch.randn((3, 16, cfg.latent_h, cfg.latent_w), generator=g, device="cuda"))
torch.cuda.synchronize()
print("ok")
