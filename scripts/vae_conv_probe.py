"""Time one VAE conv (bc_vae_conv) at decoder sizes with different epilogue
loads: out16 only / act only / res + out32 + act -- separates the
implicit-GEMM mainloop from the epilogue cost."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2511_20426_b200 import _native as N  # noqa: E402


def run(H, W, frames, cin, cout, kt, kh, kw, mode, reps=5):
    x = torch.randn((frames, H + 2, W + 2, cin), device="cuda").bfloat16()
    w = (torch.randn((cout, kt * kh * kw * cin), device="cuda") * 0.05).bfloat16()
    bias = torch.zeros(cout, device="cuda")
    gamma = torch.ones(cout, device="cuda")
    res = torch.zeros((frames, H + 2, W + 2, cout), device="cuda")
    out16 = torch.zeros((frames, H + 2, W + 2, cout), dtype=torch.bfloat16, device="cuda")
    a = N.VaeConvArgs()
    a.in_, a.w, a.bias = N.ptr(x), N.ptr(w), N.ptr(bias)
    a.H, a.W, a.n_frames, a.frame0, a.n_out_frames = H, W, frames, 2, frames - 2
    a.cin, a.cout, a.kt, a.kh, a.kw = cin, cout, kt, kh, kw
    if mode == "out16":
        a.out16 = N.ptr(out16)
    elif mode == "act":
        a.act, a.gamma, a.act_silu = N.ptr(out16), N.ptr(gamma), 1
    else:
        a.res, a.out32, a.act, a.gamma, a.act_silu = N.ptr(res), N.ptr(res), N.ptr(out16), N.ptr(gamma), 1
    sp = N.stream_ptr()
    N.check(N.lib().bc_vae_conv(a, sp), "conv")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        N.check(N.lib().bc_vae_conv(a, sp), "conv")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * kt * kh * kw * cin * cout * H * W * (frames - 2)
    return ms, fl / ms / 1e9


def main():
    if len(sys.argv) > 1:            # single case for ncu: NAME MODE
        geo = {"L3_96x96": (480, 832, 14, 96, 96, 3, 3, 3), "L2_192x192": (240, 416, 14, 192, 192, 3, 3, 3)}
        print(run(*geo[sys.argv[1]], sys.argv[2], reps=1))
        return
    out = {}
    for name, geo in {"L3_96x96": (480, 832, 14, 96, 96, 3, 3, 3), "L2_192x192": (240, 416, 14, 192, 192, 3, 3, 3),
                      "L1_384x384": (120, 208, 8, 384, 384, 3, 3, 3),
                      "L3_rs_192x96": (480, 832, 14, 192, 96, 1, 3, 3)}.items():
        for mode in ("out16", "act", "full"):
            if geo[4] > 192 and mode != "out16":
                continue
            ms, tf = run(*geo, mode)
            out[f"{name}:{mode}"] = {"ms": round(ms, 3), "tflops": round(tf, 1)}
            print(name, mode, out[f"{name}:{mode}"], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
