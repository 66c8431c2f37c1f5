"""CPU checks of the VAE decoder checker (oracle/vae.py) and of the product's
host-side VAE plan (paper_2511_20426_b200/vae.py): the same layer list and
parameter shapes, the causal-cache semantics, and the frame counts."""

import pytest
import torch
import torch.nn.functional as F

from oracle import vae as V


def _product():
    from paper_2511_20426_b200 import vae as P
    return P


@pytest.mark.parametrize("dim", [96, 32])
def test_product_layer_plan_matches_oracle(dim):
    P = _product()
    pc = P.vae_config("wan2.1", dim=dim)
    od = V.VaeDims(dim=dim)
    assert P.layer_specs(pc) == V.layer_specs(od)
    ps, os_ = P.param_shapes(pc), V.param_shapes(od)
    assert ps.keys() == os_.keys()
    for k in ps:
        assert ps[k] == os_[k], k


def test_wan21_decoder_channel_plan():
    dims, specs, last = V.layer_specs(V.VaeDims())
    assert dims == [384, 384, 384, 192, 96] and last == 96
    kinds = [s[0] for s in specs]
    assert kinds.count("res") == 14 and kinds.count("attn") == 1
    assert [s[0] for s in specs if s[0].startswith("up")] == ["up3d", "up3d", "up2d"]
    # the first ResidualBlock after each resample takes half the channels (Decoder3d: in_dim // 2)
    assert ("res", "up4", 192, 384) in specs and ("res", "up8", 192, 192) in specs and ("res", "up12", 96, 96) in specs


def test_causal_conv_cache_equals_stream():
    g = torch.Generator().manual_seed(0)
    x = torch.randn(1, 8, 7, 5, 6, generator=g)
    w = torch.randn(4, 8, 3, 3, 3, generator=g)
    b = torch.randn(4, generator=g)
    whole = V.causal_conv3d(x, w, b)
    cache = V._Cache()
    parts = [V._cconv(x[:, :, i:j], w, b, "c", cache) for i, j in ((0, 1), (1, 3), (3, 4), (4, 7))]
    assert torch.allclose(torch.cat(parts, 2), whole, atol=1e-5)
    # zero causal padding in front, symmetric spatial padding
    ref = F.conv3d(F.pad(x, [1, 1, 1, 1, 2, 0]), w, b)
    assert torch.allclose(whole, ref, atol=1e-5)


def test_rms_norm_is_channel_normalize():
    x = torch.randn(2, 6, 3, 4, 5)
    g = torch.rand(6) + 0.5
    y = V.rms_norm(x, g)
    want = x / x.norm(dim=1, keepdim=True) * 6 ** 0.5 * g.view(1, 6, 1, 1, 1)
    assert torch.allclose(y, want, atol=1e-5)


def test_stream_chunking_and_frame_counts():
    P = _product()
    d = V.VaeDims(dim=32)
    params = V.random_params(d, 5)
    z = torch.randn(16, 4, 4, 6, generator=torch.Generator().manual_seed(2))
    o = V.VaeDecoderOracle(params, d)
    whole = o.decode(z)
    o.reset()
    parts = [o.decode(z[:, :1]), o.decode(z[:, 1:3]), o.decode(z[:, 3:])]
    assert [p.shape[1] for p in parts] == [1, 8, 4]
    assert torch.allclose(torch.cat(parts, 1), whole, atol=1e-5)
    assert whole.shape == (3, 1 + 4 * 3, 32, 48)
    assert float(whole.abs().max()) <= 1.0
    cfg = P.vae_config("tiny")
    assert cfg.frames_out(3, True) == 9 and cfg.frames_out(3, False) == 12


def test_decoder_needs_device():
    """The product decoder has no CPU path: without CUDA it raises."""
    from paper_2511_20426_b200.errors import DeviceError
    P = _product()
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(DeviceError):
        P.VaeWeights.random(P.vae_config("tiny"), 1)
