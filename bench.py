#!/usr/bin/env python
"""Headline benchmark: generated frames/s of cascaded Wan2.1-1.3B-shaped
generation (BASELINE.json configs[1]) on B200, with the sequential
block-causal rollout, per-kernel roofline and the CPU reference timed beside
it.

A "step" is one complete 13-block generation (156 video frames, 480x832,
4-step schedule, 3 latent frames per block, offset 1 = deepest cascade),
i.e. one pass of the hot path -- 17 cascade iterations of the batched DiT
forward + fused renoise -- over one synthetic input (noise + prompt).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: W untimed warm-up generations, then K timed ones bracketed by a
barrier + torch.cuda.synchronize() on both sides, device time from CUDA
events on the launching stream, max over ranks.  Working set (2.6 GB bf16
weights + 11 GB KV arena) is far larger than the 126 MB L2, so no explicit
flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PROMPT = "a lighthouse in a storm"
SESSION_SEED = 20260809
WEIGHT_SEED = 7
FRAMES_PER_BLOCK = 12   # 3 latent frames x 4 video frames


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU reference / baseline (oracle port of the path, numpy fp32)
# ---------------------------------------------------------------------------

def cpu_sample_seconds(cfg, reps=1):
    """Time one bounded sample of the workload on the host cores: ONE of the
    `layers` transformer layers for ONE of the 5 entries of a steady-state
    cascade iteration (13 visible blocks = 60,840 keys, 4,680 query tokens,
    512 text tokens), numpy fp32 oracle (oracle/wan.py)."""
    import numpy as np
    from oracle import wan as wo
    d, T = cfg.model_dim, cfg.tokens_per_block
    rng = np.random.default_rng(0)

    def w(*shape, fan):
        return (rng.standard_normal(shape, dtype=np.float32) / np.sqrt(fan)).astype(np.float32)

    p = {"qkv_w": w(3 * d, d, fan=d), "qkv_b": w(3 * d, fan=50), "o_w": w(d, d, fan=d),
         "o_b": w(d, fan=50), "cq_w": w(d, d, fan=d), "cq_b": w(d, fan=50),
         "co_w": w(d, d, fan=d), "co_b": w(d, fan=50), "ffn1_w": w(cfg.ffn_dim, d, fan=d),
         "ffn1_b": w(cfg.ffn_dim, fan=50), "ffn2_w": w(d, cfg.ffn_dim, fan=cfg.ffn_dim),
         "ffn2_b": w(d, fan=50), "nq": 1 + w(d, fan=400), "nk": 1 + w(d, fan=400),
         "n3w": 1 + w(d, fan=400), "n3b": w(d, fan=50), "cnq": 1 + w(d, fan=400),
         "mod": w(6, d, fan=d)}
    X = rng.standard_normal((T, d), dtype=np.float32)
    pool_k = rng.standard_normal((12 * T, d), dtype=np.float32)
    pool_v = rng.standard_normal((12 * T, d), dtype=np.float32)
    tk = rng.standard_normal((cfg.text_len, d), dtype=np.float32)
    tv = rng.standard_normal((cfg.text_len, d), dtype=np.float32)
    cos, sin = wo.rope_tables(27, cfg.block_size, cfg.latent_height // 2, cfg.latent_width // 2)
    H = cfg.heads
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        m = p["mod"]
        xn = wo.layer_norm(X) * (1 + m[1]) + m[0]
        qkv = xn @ p["qkv_w"].T + p["qkv_b"]
        q = wo.apply_rope(wo.rms_norm(qkv[:, :d], p["nq"]).reshape(T, H, 128), cos, sin).reshape(T, d)
        k = wo.apply_rope(wo.rms_norm(qkv[:, d:2 * d], p["nk"]).reshape(T, H, 128), cos, sin).reshape(T, d)
        att = wo.attention(q, np.concatenate([pool_k, k]), np.concatenate([pool_v, qkv[:, 2 * d:]]), H)
        Xo = X + m[2] * (att @ p["o_w"].T + p["o_b"])
        xc = wo.layer_norm(Xo) * p["n3w"] + p["n3b"]
        qc = wo.rms_norm(xc @ p["cq_w"].T + p["cq_b"], p["cnq"])
        Xo = Xo + wo.attention(qc, tk, tv, H) @ p["co_w"].T + p["co_b"]
        xm = wo.layer_norm(Xo) * (1 + m[4]) + m[3]
        Xo = Xo + m[5] * (wo.gelu_tanh(xm @ p["ffn1_w"].T + p["ffn1_b"]) @ p["ffn2_w"].T + p["ffn2_b"])
        times.append(time.perf_counter() - t0)
    return times


def cpu_fps_from_sample(cfg, sample_s):
    width = min(cfg.cascade_width, cfg.num_blocks)
    iter_s = sample_s * cfg.layers * width     # one steady-state iteration emits one block
    return FRAMES_PER_BLOCK / iter_s


def cpu_sample_desc(cfg):
    return (f"1 of {cfg.layers} layers x 1 of {min(cfg.cascade_width, cfg.num_blocks)} entries of a "
            f"steady-state cascade iteration ({cfg.tokens_per_block} query tokens, 13 visible blocks = "
            f"{13 * cfg.tokens_per_block} keys, {cfg.text_len} text tokens), numpy fp32 oracle; "
            f"fps = 12 frames / (sample x {cfg.layers * min(cfg.cascade_width, cfg.num_blocks)})")


TOY_CFG1 = dict(layers=4, latent_dim=256, heads=2, head_dim=128, cond_dim=256, total_frames=18,
                offset=1, window_blocks=7, sink_blocks=1, attention_mode="bidirectional")


def toy_config1_times(bc):
    """BASELINE configs[0]: the reference toy model (L4, D256, 6 blocks, o=1,
    bidirectional) through run_cascade on the device (fp64 kernels) and through
    the same engine driven by the numpy oracle forward on the host."""
    import torch
    from paper_2511_20426_b200 import engine
    from oracle.loop import oracle_runtime
    cfg1 = bc.CascadeConfig(**TOY_CFG1).validate()
    w = bc.init_model(WEIGHT_SEED, cfg1.layers, cfg1.heads, cfg1.latent_dim, cfg1.cond_dim)

    def med(f, n):
        ts = []
        for _ in range(n):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts) * 1e3
    gpu = bc.run_cascade(cfg1, "a red cube", weights=w)
    gpu_ms = med(lambda: bc.run_cascade(cfg1, "a red cube", weights=w), 5)
    gpu_seq_ms = med(lambda: bc.run_sequential_reference(cfg1, "a red cube", weights=w), 5)
    orig = engine._runtime_for
    engine._runtime_for = oracle_runtime
    try:
        cpu = bc.run_cascade(cfg1, "a red cube", weights=w)
        cpu_ms = med(lambda: bc.run_cascade(cfg1, "a red cube", weights=w), 5)
        cpu_seq_ms = med(lambda: bc.run_sequential_reference(cfg1, "a red cube", weights=w), 5)
    finally:
        engine._runtime_for = orig
    import numpy as np
    rel = max(float(np.linalg.norm(gpu.outputs[b] - cpu.outputs[b]) / np.linalg.norm(cpu.outputs[b]))
              for b in cpu.outputs)
    return {"workload": "reference toy model, L4 D256 2x128 heads, 6 blocks (18 frames), o=1, bidirectional",
            "device_fp64_ms_per_run": round(gpu_ms, 2), "oracle_cpu_ms_per_run": round(cpu_ms, 2),
            "sequential_device_fp64_ms_per_run": round(gpu_seq_ms, 2),
            "sequential_oracle_cpu_ms_per_run": round(cpu_seq_ms, 2), "median_of": 5,
            "max_block_rel_l2_vs_oracle": rel}


def noise_generation_report(cfg):
    """host noise generation reported separately.  Every (block,
    pass) draw of one run (Philox4x64 + numpy's ziggurat, fp32), by the
    native multi-threaded generator the e2e path uses, vs numpy itself for one
    block-pass (the reference's GIL-bound path, core.py:170-186)."""
    import numpy as np
    from paper_2511_20426_b200 import _native as N
    from paper_2511_20426_b200.wan import run_noise_keys
    keys = run_noise_keys(cfg)
    S, D = cfg.block_size, cfg.latent_dim
    threads = max(1, os.cpu_count() or 1)
    out = np.empty((len(keys), S, D), dtype=np.float32)
    tasks = [(SESSION_SEED, 0, (b, p, b * S + i, 0), out[k, i]) for k, (b, p) in enumerate(keys) for i in range(S)]
    N.run_noise_tasks(tasks, 1, threads)  # warm-up (page-in)
    t0 = time.perf_counter()
    N.run_noise_tasks(tasks, 1, threads)
    native_s = time.perf_counter() - t0
    stream = __import__("paper_2511_20426_b200").NoiseStream(SESSION_SEED, D)
    t0 = time.perf_counter()
    ref = np.stack([stream.draw(0, 1, i) for i in range(S)])
    numpy_s = time.perf_counter() - t0
    if not np.array_equal(ref.astype(np.float32), out[keys.index((0, 1))]):
        raise RuntimeError("native noise differs from numpy's draws")
    return {"block_passes_per_run": len(keys), "native_ms_per_run": round(native_s * 1e3, 2),
            "native_ms_per_block_pass": round(native_s * 1e3 / len(keys), 3), "threads": threads,
            "numpy_ms_per_block_pass": round(numpy_s * 1e3, 2),
            "bytes_per_run": int(out.nbytes), "bit_identical_to_numpy": True}


def metric_name(args):
    return f"generated frames/sec (cascaded, Wan2.1-{args.preset.upper()}-shaped, 480x832)"


def workload_config(args, cfg, parallelism):
    return {"workload": f"wan2.1-{args.preset} cascade o=1, {cfg.num_blocks} blocks "
                        f"({cfg.num_blocks * FRAMES_PER_BLOCK} frames), 480x832, 4-step, "
                        f"3 latent frames/block, bidirectional, W=7 sink={args.sink}"
                        + (f", cascade prompt switch every {args.switch_every} blocks"
                           if args.switch_every else ""),
            "model": f"wan2.1-{args.preset}-shaped", "global_batch": 1,
            "seq_len": cfg.tokens_per_block, "parallelism": parallelism,
            "l2": "working set (weights + KV arena) >> 126 MB L2; no flush"}


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count()
    for _ in range(args.warmup):
        cpu_sample_seconds(cfg)
    times = [cpu_sample_seconds(cfg)[0] for _ in range(args.steps)]
    per = statistics.mean(times)
    fps = cpu_fps_from_sample(cfg, per)
    line = {
        "impl": "reference", "metric": metric_name(args),
        "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (random-init weights, N(0,1) activations)",
        "config": workload_config(args, cfg, f"temporal{world}"),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port",
                         "sample": cpu_sample_desc(cfg)},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, cfg):
    import torch
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import _native as N
    from paper_2511_20426_b200.metrics import end_to_end_fps, streaming_fps
    from paper_2511_20426_b200.wan import ResidentNoiseFeed, WanWeights, run_noise_keys

    world, rank, local = dist_env()
    # BC_FORCE_DEVICE / BC_DIST_BACKEND: test hooks to run the multi-rank
    # bench with several ranks on one GPU over gloo (NCCL refuses duplicate
    # GPUs); the driver's runs use one GPU per rank and NCCL
    dev = int(os.environ.get("BC_FORCE_DEVICE", local))
    backend = os.environ.get("BC_DIST_BACKEND", "nccl")
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend)

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    weights = WanWeights.random(cfg, WEIGHT_SEED)
    seq_cfg = bc.with_fields(cfg, offset=cfg.passes)
    feed = ResidentNoiseFeed(SESSION_SEED, cfg, run_noise_keys(cfg))

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    switches = [bc.SwitchSpec(f"{PROMPT}, scene {k}", "cascade", at_block=k)
                for k in range(args.switch_every, cfg.num_blocks, args.switch_every)] \
        if args.switch_every else []

    def one_run(c=cfg, noise=feed):
        return bc.run_cascade(c, PROMPT, session_seed=SESSION_SEED, weights=weights, noise_feed=noise,
                              switches=switches)

    for _ in range(args.warmup):
        one_run()
    N.profile_collect()
    # ---- timed region: device-resident inputs ----
    N.profile_enable(True)
    launches0 = N.launch_count()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        ev0.record()
        runs = [one_run() for _ in range(args.steps)]
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    launches = N.launch_count() - launches0
    prof = N.profile_collect()
    N.profile_enable(False)
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    # temporal parallelism: all ranks cooperate on ONE video (strong scaling)
    frames = cfg.num_blocks * FRAMES_PER_BLOCK
    value = frames * args.steps / (ms / 1e3)
    stream_fps = statistics.mean(streaming_fps(r.trace, clock="wall") for r in runs)

    # ---- e2e through the public API with host buffers (noise H2D, outputs D2H) ----
    # (measured right after the device-resident runs, under the same thermal /
    # power state; its own clock samples are reported as clocks_e2e)
    # one untimed end-to-end run first: the host-noise path's pinned staging
    # buffers and first-touch costs are warm-up, not steady state
    bc.run_cascade(cfg, PROMPT, session_seed=SESSION_SEED, weights=weights, switches=switches)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clocks_e2e:
        t0 = time.perf_counter()
        e2e_runs = [bc.run_cascade(cfg, PROMPT, session_seed=SESSION_SEED, weights=weights,
                                   switches=switches) for _ in range(args.steps)]
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
    e2e_s = max_over_ranks(e2e_s)
    e2e_value = frames * args.steps / e2e_s
    # ---- sequential block-causal rollout, same weights / inputs ----
    seq_e2e = seq_stream = None
    if not args.no_seq:
        for _ in range(2):
            seq = bc.run_sequential_reference(seq_cfg, PROMPT, session_seed=SESSION_SEED,
                                              weights=weights, noise_feed=feed)
        seq_e2e = end_to_end_fps(seq.trace)
        seq_stream = streaming_fps(seq.trace, clock="wall")

    # ---- prompt switch at block 8: cascade mode (product: text K/V swap only)
    # vs the KV-recache baseline (paper: ~200 ms stall) ----
    switch = None
    if world == 1 and not args.no_switch and cfg.num_blocks > 9:
        switch = {"at_block": 8}
        for mode in ("cascade", "recache"):
            sw = [bc.SwitchSpec(f"{PROMPT}, new scene", mode, at_block=8)]
            r = bc.run_cascade(cfg, PROMPT, session_seed=SESSION_SEED, weights=weights,
                               noise_feed=feed, switches=sw)
            evs = r.trace.events
            k = next(i for i, e in enumerate(evs) if e.switch is not None)
            prev = evs[k - 1].wall_clock if k else 0.0
            stall_ms = (evs[k].wall_clock - prev - evs[k].wall_seconds) * 1e3
            nxt = next(e for e in evs[k:] if e.emitted_block is not None)
            switch[mode] = {"extra_passes": r.switch_events[0].extra_passes,
                            "stall_ms": round(stall_ms, 3),
                            "pool_blocks": evs[k].pool_blocks,
                            "fps_next_block": round(nxt.emitted_video_frames /
                                                    (nxt.wall_clock - prev), 2),
                            "e2e_fps": end_to_end_fps(r.trace)}

    # ---- the reference's own CPU-runnable case (BASELINE configs[0]): the toy
    # model of the reference package, fp64 on the device, vs the oracle port
    # of it on the host (the reference code itself is not on the box) ----
    toy = noise = None
    if world == 1 and not args.no_cpu:
        toy = toy_config1_times(bc)
        noise = noise_generation_report(cfg)

    S = cfg.block_size
    lat_bytes = S * cfg.latent_dim * 4
    h2d = len(run_noise_keys(cfg)) * lat_bytes + cfg.text_len * cfg.text_dim * 4
    d2h = cfg.num_blocks * lat_bytes

    if rank != 0:
        return
    peaks, peak_kind = _peaks()
    dom = max(("self_attention", "cross_attention", "gemm"), key=lambda k: prof[k][0])
    dom_ms, dom_flops, _, dom_n = prof[dom]
    achieved = dom_flops / (dom_ms / 1e3) / 1e12 if dom_ms > 0 else None
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(dom)
    total_prof_ms = sum(v[0] for v in prof.values())
    kernels = {k: {"ms": round(v[0], 3), "launches": v[3],
                   "tflops": round(v[1] / (v[0] / 1e3) / 1e12, 1) if v[0] > 0 and v[1] > 0 else None,
                   "gbs": round(v[2] / (v[0] / 1e3) / 1e9, 1) if v[0] > 0 and v[2] > 0 else None,
                   "share": round(v[0] / total_prof_ms, 4) if total_prof_ms else None}
               for k, v in prof.items()}
    # CPU baseline on a bounded sample (rank 0, N=1 only)
    cpu = None
    if world == 1 and not args.no_cpu:
        samp = cpu_sample_seconds(cfg, reps=1)[0]
        cpu = {"value": cpu_fps_from_sample(cfg, samp), "unit": "frames/s", "cores": os.cpu_count(),
               "kind": "port", "sample": cpu_sample_desc(cfg), "sample_seconds": samp}
    line = {
        "metric": metric_name(args),
        "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": f"synthetic (random-init Wan2.1-{args.preset.upper()}-shaped weights, counter-keyed N(0,1) "
                "noise, hash-expanded 512x4096 text states)",
        "config": workload_config(args, cfg, f"temporal{world}"),
        "streaming_fps": stream_fps,
        "sequential": {"e2e_fps": seq_e2e, "streaming_fps": seq_stream},
        "cascade_over_sequential_streaming": stream_fps / seq_stream if seq_stream else None,
        "prompt_switch": switch,
        "config1_toy": toy,
        "noise_generation": noise,
        "roofline": {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak if achieved else None,
                     "traffic": traffic, "peak_kind": f"{peak_kind} bf16 sustained",
                     "launches": dom_n, "share_of_step": kernels[dom]["share"]},
        "kernels": kernels,
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "clocks_e2e": clocks_e2e.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--preset", default="1.3b")
    ap.add_argument("--blocks", type=int, default=13)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--sink", type=int, default=1, help="sink blocks (LongLive-style: 0)")
    ap.add_argument("--switch-every", type=int, default=0,
                    help="cascade-mode prompt switch every N blocks (LongLive-style config 5)")
    ap.add_argument("--no-seq", action="store_true", help="skip the sequential rollout")
    ap.add_argument("--no-switch", action="store_true",
                    help="skip the cascade-vs-recache prompt-switch measurement")
    args = ap.parse_args()
    from paper_2511_20426_b200 import wan_config
    cfg = wan_config(args.preset, total_frames=3 * args.blocks, offset=1,
                     attention_mode="bidirectional", window_blocks=7, sink_blocks=args.sink)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
