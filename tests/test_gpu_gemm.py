"""tcgen05 GEMM (csrc/gemm.cu) vs a plain PyTorch fp32 reference of the same
op on the same bf16 inputs.  Tolerances: fp32 outputs rel-L2 <= 1e-5
(accumulation order only); bf16 outputs rel-L2 <= 4e-3 (one bf16 rounding)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2511_20426_b200 import _native as N


def gemm(A, B, C, mode, bias=None, gate=None, gate_stride=0, rows_per_gate=1, bn=0, cg=0):
    M, K = A.shape
    Nn = B.shape[0]
    N.check(N.lib().bc_gemm_bf16(N.ptr(A), N.ptr(B), N.ptr(C), M, Nn, K,
                                 mode | width_bits(bn) | (cg << 16),
                                 N.ptr(bias), N.ptr(gate), gate_stride, rows_per_gate,
                                 N.stream_ptr()), "gemm")


def width_bits(bn):
    """Forced tile width: bits 8-15 in units of 64 columns, or of 32 with bit 18."""
    return ((bn // 64) << 8) if bn % 64 == 0 else ((bn // 32) << 8) | (1 << 18)


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


SHAPES = [(128, 256, 64), (300, 128, 128), (4680, 1536, 1536), (1000, 768, 256),
          (192, 64, 256), (4680, 4608, 1536), (512, 1536, 4096), (9360, 8960, 1536)]


@pytest.mark.parametrize("M,Nn,K", SHAPES)
@pytest.mark.parametrize("bn,cg", [(0, 0), (64, 1), (128, 1), (256, 1), (256, 2), (224, 2), (192, 2)])
def test_gemm_modes(M, Nn, K, bn, cg):
    """cg = 2: tcgen05.mma.cta_group::2 CTA pairs (256 x 256 / 224 / 192
    tiles); 224-wide tiles end in a ragged, masked column tile when 224 does
    not divide N."""
    if bn and bn != 224 and Nn % bn:
        pytest.skip("tile width does not divide N")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + Nn + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(Nn, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(Nn, device="cuda", generator=g)
    ref = A.float() @ B.float().T + bias
    C = torch.empty(M, Nn, device="cuda", dtype=torch.float32)
    gemm(A, B, C, 2, bias, bn=bn, cg=cg)
    assert rel(C, ref) < 1e-5
    Cb = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    gemm(A, B, Cb, 0, bias, bn=bn, cg=cg)
    assert rel(Cb, ref) < 4e-3
    gemm(A, B, Cb, 1, bias, bn=bn, cg=cg)
    assert rel(Cb, torch.nn.functional.gelu(ref, approximate="tanh")) < 4e-3
    rows_per_gate = 97
    groups = (M + rows_per_gate - 1) // rows_per_gate
    gate = torch.randn(groups, Nn, device="cuda", generator=g)
    X = torch.randn(M, Nn, device="cuda", generator=g)
    want = X + gate.repeat_interleave(rows_per_gate, 0)[:M] * ref
    gemm(A, B, X, 3, bias, gate, Nn, rows_per_gate, bn=bn, cg=cg)
    assert rel(X, want) < 1e-5


def test_gemm_rejects_bad_shapes():
    A = torch.zeros(128, 96, device="cuda", dtype=torch.bfloat16)
    B = torch.zeros(128, 96, device="cuda", dtype=torch.bfloat16)
    C = torch.zeros(128, 128, device="cuda")
    with pytest.raises(Exception):
        gemm(A, B, C, 2)


@pytest.mark.parametrize("M,Nn,K", [(4680, 1536, 1536), (600, 512, 8960), (9360, 4608, 1536)])
def test_gemm_tilings_bitwise_equal(M, Nn, K):
    """Every tiling (64/128/256 columns, single CTA or CTA pair) runs the K
    loop in the same order, so the fp32 outputs are bit-identical -- the
    runtime's automatic tile choice can never change a result."""
    g = torch.Generator(device="cuda").manual_seed(M + Nn + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(Nn, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(Nn, device="cuda", generator=g)
    outs = []
    for bn, cg in ((64, 1), (128, 1), (256, 1), (256, 2), (224, 2), (192, 2), (0, 0)):
        if bn != 224 and Nn % (bn or 64):
            continue
        C = torch.empty(M, Nn, device="cuda")
        gemm(A, B, C, 2, bias=bias, bn=bn, cg=cg)
        outs.append(C)
    for C in outs[1:]:
        assert torch.equal(C, outs[0])


@pytest.mark.parametrize("M,Nn,K", [(4680, 1536, 1536), (777, 1536, 8960), (300, 768, 256)])
def test_gemm_residual_tilings_bitwise_equal(M, Nn, K):
    """The gated-residual epilogue (C read and written in place through TMA
    boxes) gives bit-identical C for every tiling, with and without the
    bias / gate, including a ragged last row tile."""
    g = torch.Generator(device="cuda").manual_seed(M * 3 + Nn + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(Nn, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(Nn, device="cuda", generator=g)
    rows_per_gate = 211
    gate = torch.randn((M + rows_per_gate - 1) // rows_per_gate, Nn, device="cuda", generator=g)
    X0 = torch.randn(M, Nn, device="cuda", generator=g)
    ref = A.float() @ B.float().T
    for use_bias, use_gate in ((True, True), (False, False)):
        want = X0 + (gate.repeat_interleave(rows_per_gate, 0)[:M] if use_gate else 1.0) * (ref + (bias if use_bias else 0.0))
        outs = []
        for bn, cg in ((64, 1), (128, 1), (256, 1), (256, 2), (224, 2), (192, 2), (0, 0)):
            if bn != 224 and Nn % (bn or 64):
                continue
            X = X0.clone()
            gemm(A, B, X, 3, bias if use_bias else None, gate if use_gate else None, Nn, rows_per_gate, bn=bn, cg=cg)
            outs.append(X)
        assert rel(outs[0], want) < 1e-5
        for X in outs[1:]:
            assert torch.equal(X, outs[0])

