"""VAE decode on the device against the checker.

* the tcgen05 implicit-GEMM causal conv (csrc/vae.cu) against torch fp32
  ``F.conv3d`` on the SAME bf16 operands, for every tap shape and unit
  shape the decoder uses, with each fused epilogue (bias, residual, fp32 /
  bf16 stores, RMS-norm(+SiLU) of the next layer's input, clamped video);
* the streaming decoder (paper_2511_20426_b200/vae.py) against the fp32
  Wan2.1 VAE restatement (oracle/vae.py, frame-at-a-time with Wan's feature
  caches), block after block, on the tiny geometry and at the full
  480x832 Wan2.1 geometry.

Tolerances: conv kernel rel-L2 <= 1e-5 (same bf16 operands, fp32
accumulation; only the summation order differs); decoded video rel-L2 <=
VIDEO_TOL per block (bf16 activations between ~40 layers vs fp32).
"""

import json
import os

import pytest

pytestmark = pytest.mark.gpu

VIDEO_TOL = 1e-2
CONV_TOL = 1e-5
REPORT = {}


def rel(a, b):
    a = a.double().flatten()
    b = b.double().flatten().to(a.device)
    return float((a - b).norm() / b.norm())


@pytest.fixture(scope="module", autouse=True)
def report():
    yield
    path = os.environ.get("BC_VAE_REPORT")
    if path and REPORT:
        with open(path, "w") as fh:
            json.dump(REPORT, fh, indent=1, sort_keys=True)


def _padded(torch, T, H, W, C, gen, scale=1.0):
    x = torch.zeros((T, H + 2, W + 2, C), dtype=torch.bfloat16, device="cuda")
    x[:, 1:H + 1, 1:W + 1] = (scale * torch.randn((T, H, W, C), generator=gen, device="cuda")).bfloat16()
    return x


@pytest.mark.parametrize("kt,kh,kw,cin,cout,H,W,frames", [
    (3, 3, 3, 64, 192, 9, 21, 5),      # CK 64, 2 row tiles x 192 columns
    (3, 3, 3, 384, 384, 6, 13, 4),     # 2 column groups
    (3, 3, 3, 32, 384, 5, 11, 5),      # CK 32 (conv1 with padded z channels)
    (3, 3, 3, 96, 96, 17, 40, 4),      # 4 row tiles x 96 columns (top level)
    (3, 3, 3, 96, 16, 8, 33, 3),       # head (16 padded output channels)
    (1, 3, 3, 384, 192, 10, 26, 4),    # Resample conv2d
    (3, 1, 1, 384, 768, 5, 9, 5),      # upsample3d time conv
    (1, 1, 1, 192, 384, 7, 12, 3),     # shortcut
    (1, 1, 1, 384, 1152, 6, 10, 3),    # to_qkv
])
def test_vae_conv_matches_torch(kt, kh, kw, cin, cout, H, W, frames):
    import torch
    import torch.nn.functional as F
    from paper_2511_20426_b200 import _native as N
    from oracle.wan_torch import exact_fp32

    g = torch.Generator(device="cuda")
    g.manual_seed(cin * 7 + cout)
    x = _padded(torch, frames, H, W, cin, g)
    w = (torch.randn((cout, cin, kt, kh, kw), generator=g, device="cuda") / (cin * kt * kh * kw) ** 0.5).bfloat16()
    bias = 0.1 * torch.randn(cout, generator=g, device="cuda")
    res = torch.randn((frames, H + 2, W + 2, cout), generator=g, device="cuda")
    gamma = 1 + 0.1 * torch.randn(cout, generator=g, device="cuda")
    wdev = w.permute(0, 2, 3, 4, 1).reshape(cout, -1).contiguous()
    out32 = torch.zeros_like(res)
    out16 = torch.zeros((frames, H + 2, W + 2, cout), dtype=torch.bfloat16, device="cuda")
    act = torch.zeros_like(out16)
    res0 = res.clone()
    frame0 = kt - 1 if kt == 3 else 1
    T = frames - frame0
    a = N.VaeConvArgs()
    a.in_, a.w, a.bias = N.ptr(x), N.ptr(wdev), N.ptr(bias)
    a.H, a.W, a.n_frames, a.frame0, a.n_out_frames = H, W, frames, frame0, T
    a.cin, a.cout, a.kt, a.kh, a.kw = cin, cout, kt, kh, kw
    a.res, a.out32, a.out16 = N.ptr(res), N.ptr(out32), N.ptr(out16)
    fuse_norm = cout <= 192 or cout % 192 != 0   # the norm needs the whole row in one unit
    if fuse_norm:
        a.act, a.gamma, a.act_silu = N.ptr(act), N.ptr(gamma), 1
    N.check(N.lib().bc_vae_conv(a, N.stream_ptr()), "bc_vae_conv")
    torch.cuda.synchronize()
    with exact_fp32():
        xin = x[:, 1:H + 1, 1:W + 1].float().permute(3, 0, 1, 2).unsqueeze(0)   # [1, C, T, H, W]
        pt, ph, pw = kt - 1, (kh - 1) // 2, (kw - 1) // 2
        ref = F.conv3d(F.pad(xin, [pw, pw, ph, ph, 0, 0]), w.float(), bias)      # frames frame0-(kt-1) ..
        ref = ref[0].permute(1, 2, 3, 0)                                          # [T', H, W, cout]
        ref = ref[frame0 - pt:frame0 - pt + T] + res0[frame0:frame0 + T, 1:H + 1, 1:W + 1]
    got = out32[frame0:frame0 + T, 1:H + 1, 1:W + 1]
    e = rel(got, ref)
    REPORT[f"conv_{kt}{kh}{kw}_{cin}x{cout}"] = e
    assert e < CONV_TOL, e
    assert rel(out16[frame0:frame0 + T, 1:H + 1, 1:W + 1].float(), ref) < 5e-3
    # border and frames outside the output range untouched
    assert float(out32[:, 0].abs().max()) == 0.0 and float(out32[:, :, -1].abs().max()) == 0.0
    if frame0 > 0:
        assert float(out32[:frame0].abs().max()) == 0.0
    if fuse_norm:
        n = torch.nn.functional.normalize(ref, dim=-1) * cout ** 0.5 * gamma
        want = torch.nn.functional.silu(n)
        assert rel(act[frame0:frame0 + T, 1:H + 1, 1:W + 1].float(), want) < 5e-3


def test_vae_conv_video_epilogue():
    import torch
    import torch.nn.functional as F
    from paper_2511_20426_b200 import _native as N
    from oracle.wan_torch import exact_fp32

    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    H, W, frames, cin = 12, 20, 5, 32
    x = _padded(torch, frames, H, W, cin, g, scale=2.0)
    w = torch.zeros((16, cin, 3, 3, 3), device="cuda")
    w[:3] = torch.randn((3, cin, 3, 3, 3), generator=g, device="cuda") / (cin * 27) ** 0.5
    w = w.bfloat16()
    bias = torch.zeros(16, device="cuda")
    video = torch.full((3, 3, H, W), 7.0, device="cuda")
    a = N.VaeConvArgs()
    a.in_, a.w, a.bias = N.ptr(x), N.ptr(w.permute(0, 2, 3, 4, 1).reshape(16, -1).contiguous()), N.ptr(bias)
    a.H, a.W, a.n_frames, a.frame0, a.n_out_frames = H, W, frames, 2, 3
    a.cin, a.cout, a.kt, a.kh, a.kw = cin, 16, 3, 3, 3
    a.video, a.video_channels = N.ptr(video), 3
    keep = a.w
    N.check(N.lib().bc_vae_conv(a, N.stream_ptr()), "bc_vae_conv")
    torch.cuda.synchronize()
    with exact_fp32():
        xin = x[:, 1:H + 1, 1:W + 1].float().permute(3, 0, 1, 2).unsqueeze(0)
        ref = F.conv3d(F.pad(xin, [1, 1, 1, 1, 0, 0]), w.float()[:3])[0].permute(1, 0, 2, 3).clamp(-1, 1)
    assert keep
    assert rel(video, ref) < CONV_TOL


def _decode_vs_oracle(cfg, n_blocks, seed, tol, key):
    import torch
    from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights
    from oracle import vae as V
    from oracle.wan_torch import exact_fp32

    wts = VaeWeights.random(cfg, seed)
    dec = VaeDecoder(wts)
    dec.reset()
    dims = V.VaeDims(dim=cfg.dim, z_dim=cfg.z_dim, dim_mult=cfg.dim_mult, num_res_blocks=cfg.num_res_blocks,
                     temperal_upsample=cfg.temporal_upsample)
    orc = V.VaeDecoderOracle(wts.host_params(device="cuda"), dims)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed + 1)
    errs = []
    for b in range(n_blocks):
        z = torch.randn((cfg.block_size, cfg.z_dim, cfg.latent_h, cfg.latent_w), generator=g, device="cuda")
        got = dec.decode_block(z)
        dec.wait()
        with exact_fp32():
            ref = orc.decode(z.permute(1, 0, 2, 3))                       # [3, n, 8h, 8w]
        ref = ref.permute(1, 0, 2, 3)
        assert got.shape == ref.shape, (got.shape, ref.shape)
        assert got.shape[0] == cfg.frames_out(cfg.block_size, b == 0)
        errs.append(rel(got, ref))
    REPORT[key] = errs
    assert max(errs) < tol, errs
    return dec


def test_vae_decode_tiny_stream():
    from paper_2511_20426_b200.vae import vae_config
    _decode_vs_oracle(vae_config("tiny"), 3, 21, VIDEO_TOL, "decode_tiny_rel_l2_per_block")


def test_vae_decode_reset_restarts_stream():
    import torch
    from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights, vae_config

    cfg = vae_config("tiny")
    dec = VaeDecoder(VaeWeights.random(cfg, 4))
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    zs = [torch.randn((cfg.block_size, cfg.z_dim, cfg.latent_h, cfg.latent_w), generator=g, device="cuda")
          for _ in range(2)]
    def run():
        dec.reset()
        outs = [dec.decode_block(z) for z in zs]
        dec.wait()
        return [o.clone() for o in outs]
    a = run()
    b = run()
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x, y)            # deterministic, caches fully reset


def test_vae_decode_wan_geometry():
    from paper_2511_20426_b200.vae import vae_config
    _decode_vs_oracle(vae_config("wan2.1"), 2, 33, VIDEO_TOL, "decode_wan2.1_480x832_rel_l2_per_block")


def test_vae_decode_lane_in_run_cascade():
    """run_cascade(decoder=...) decodes every emitted block on the decoder's
    stream (the reference's decode lane, engine.py:151-158, made real): the
    videos equal an independent decode of the run's outputs in emission
    order, decode stamps follow emissions, and the decode-inclusive
    streaming FPS is defined."""
    import numpy as np
    import torch
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import metrics
    from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights, vae_config
    from paper_2511_20426_b200.wan import WanWeights

    cfg = bc.wan_config("tiny", total_frames=27)
    vcfg = vae_config("tiny", latent_h=cfg.latent_height, latent_w=cfg.latent_width)
    vw = VaeWeights.random(vcfg, 3)
    res = bc.run_cascade(cfg, "a lighthouse", weights=WanWeights.random(cfg, 7), decoder=VaeDecoder(vw))
    assert sorted(res.videos) == list(range(cfg.num_blocks))
    ref = VaeDecoder(vw)
    ref.reset()
    for k, b in enumerate(res.emitted_order):
        z = torch.from_numpy(res.outputs[b].astype(np.float32).reshape(
            cfg.block_size, cfg.latent_channels, cfg.latent_height, cfg.latent_width)).cuda()
        want = ref.decode_block(z)
        ref.wait()
        got = res.videos[b]
        assert got.shape == (vcfg.frames_out(cfg.block_size, k == 0), 3, vcfg.video_h, vcfg.video_w)
        assert torch.equal(got, want), b
    ems = res.trace.emissions
    for ev in ems:
        assert ev.decode_start is not None and ev.decode_done >= ev.decode_start >= 0.0
        assert ev.decode_done >= ev.wall_clock - 1e-6
    done = [ev.decode_done for ev in ems]
    assert done == sorted(done)
    assert metrics.streaming_fps(res.trace, clock="decoded") > 0.0
    # a block cannot be decoded before it was emitted: decoded e2e FPS is at
    # most the frames over the last EMISSION time (the run's wall clock also
    # holds the trailing cache passes, so it can end after the last decode)
    frames = sum(ev.emitted_video_frames for ev in ems)
    assert metrics.end_to_end_fps(res.trace, clock="decoded") <= frames / ems[-1].wall_clock + 1e-9
