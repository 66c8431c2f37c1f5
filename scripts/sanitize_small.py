"""Small launches of every device kernel family for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2511_20426_b200 as bc
from paper_2511_20426_b200 import _native as N
from paper_2511_20426_b200.wan import WanWeights

# GEMM, all epilogues, ragged M
A = torch.randn(300, 256, device="cuda").bfloat16(); B = torch.randn(256, 256, device="cuda").bfloat16()
for mode, dt in ((0, torch.bfloat16), (1, torch.bfloat16), (2, torch.float32), (3, torch.float32)):
    C = torch.zeros(300, 256, device="cuda", dtype=dt)
    g = torch.ones(4, 256, device="cuda")
    N.check(N.lib().bc_gemm_bf16(N.ptr(A), N.ptr(B), N.ptr(C), 300, 256, 256, mode, 0,
                                 N.ptr(g) if mode == 3 else 0, 256, 100, N.stream_ptr()), "gemm")
# CTA-pair GEMM (cta_group::2, 256-row tiles), ragged M, all epilogues
A2 = torch.randn(600, 256, device="cuda").bfloat16(); B2 = torch.randn(512, 256, device="cuda").bfloat16()
for mode, dt in ((0, torch.bfloat16), (1, torch.bfloat16), (2, torch.float32), (3, torch.float32)):
    C = torch.zeros(600, 512, device="cuda", dtype=dt)
    g = torch.ones(6, 512, device="cuda")
    N.check(N.lib().bc_gemm_bf16(N.ptr(A2), N.ptr(B2), N.ptr(C), 600, 512, 256, mode | (4 << 8) | (2 << 16), 0,
                                 N.ptr(g) if mode == 3 else 0, 512, 100, N.stream_ptr()), "gemm pair")
# 192-column CTA-pair tiles (N = 384), ragged M
B3 = torch.randn(384, 256, device="cuda").bfloat16()
for mode, dt in ((0, torch.bfloat16), (3, torch.float32)):
    C = torch.zeros(600, 384, device="cuda", dtype=dt)
    g = torch.ones(6, 384, device="cuda")
    N.check(N.lib().bc_gemm_bf16(N.ptr(A2), N.ptr(B3), N.ptr(C), 600, 384, 256, mode | (3 << 8) | (2 << 16), 0,
                                 N.ptr(g) if mode == 3 else 0, 384, 100, N.stream_ptr()), "gemm pair 192")
# attention, ragged q/kv
T, H = 200, 2
arena = torch.randn(4, 2, T, H * 128, device="cuda").bfloat16()
q = torch.randn(2 * T, H * 128, device="cuda").bfloat16(); out = torch.empty_like(q)
b = N.make_batch(3, [0, 1], [0.0, 0.0], [0, 1], [[0, 1], [0, 1, 2, 3]])
mat = T * H * 128
N.check(N.lib().bc_attention_paged(N.ptr(q), N.ptr(arena), N.ptr(arena) + mat * 2, 2 * mat, T, b, T, H,
                                   N.ptr(out), N.stream_ptr()), "attn")
# tiny Wan cascade (all kernels incl. head update) + toy
cfg = bc.wan_config("tiny", total_frames=9)
bc.run_cascade(cfg, "p", weights=WanWeights.random(cfg, 1))
bc.run_cascade(bc.CascadeConfig(total_frames=9).validate(), "p")
# multi-rank device path (row partition, 3 emulated ranks: peer copies, flags,
# stream-memop waits, Y exchange) and the recache baseline
from paper_2511_20426_b200 import distributed
distributed.EMULATE = True
os.environ["BC_TEMPORAL_SHARD"] = "rows"
bc.run_cascade(bc.with_fields(cfg, workers=3), "p", weights=WanWeights.random(cfg, 1))
distributed.EMULATE = False
cfg12 = bc.wan_config("tiny", total_frames=12)
bc.run_cascade(cfg12, "p", weights=WanWeights.random(cfg12, 1),
               switches=[bc.SwitchSpec("q", "recache", at_block=2)])
torch.cuda.synchronize()
print("sanitize workload done")
