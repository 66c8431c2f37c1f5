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

def blas_threads():
    """Threads numpy's BLAS runs with (threadpoolctl), else the core count."""
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        if n and n[0]:
            return int(n[0])
    except Exception:
        pass
    return os.cpu_count() or 1


class CpuLayerSample:
    """One transformer layer of ONE entry with ``vis_frames`` visible latent
    frames (4,680 query tokens at 480x832; pool + own keys; 512 text
    tokens), numpy fp32 oracle (oracle/wan.py), timed on the host cores.
    Random activations / weights of the layer's shapes (built once)."""

    def __init__(self, cfg, max_vis_frames=39):
        import numpy as np
        self.cfg = cfg
        d, T = cfg.model_dim, cfg.tokens_per_block
        rng = np.random.default_rng(0)

        def w(*shape, fan):
            return (rng.standard_normal(shape, dtype=np.float32) / np.sqrt(fan)).astype(np.float32)

        self.p = {"qkv_w": w(3 * d, d, fan=d), "qkv_b": w(3 * d, fan=50), "o_w": w(d, d, fan=d),
                  "o_b": w(d, fan=50), "cq_w": w(d, d, fan=d), "cq_b": w(d, fan=50),
                  "co_w": w(d, d, fan=d), "co_b": w(d, fan=50), "ffn1_w": w(cfg.ffn_dim, d, fan=d),
                  "ffn1_b": w(cfg.ffn_dim, fan=50), "ffn2_w": w(d, cfg.ffn_dim, fan=cfg.ffn_dim),
                  "ffn2_b": w(d, fan=50), "nq": 1 + w(d, fan=400), "nk": 1 + w(d, fan=400),
                  "n3w": 1 + w(d, fan=400), "n3b": w(d, fan=50), "cnq": 1 + w(d, fan=400),
                  "mod": w(6, d, fan=d)}
        self.X = rng.standard_normal((T, d), dtype=np.float32)
        pool_tokens = max(0, max_vis_frames // cfg.block_size - 1) * T
        self.pool_k = rng.standard_normal((pool_tokens, d), dtype=np.float32)
        self.pool_v = rng.standard_normal((pool_tokens, d), dtype=np.float32)
        self.tk = rng.standard_normal((cfg.text_len, d), dtype=np.float32)
        self.tv = rng.standard_normal((cfg.text_len, d), dtype=np.float32)

    def seconds(self, vis_frames):
        import numpy as np
        from oracle import wan as wo
        cfg, p = self.cfg, self.p
        d, T, H = cfg.model_dim, cfg.tokens_per_block, cfg.heads
        npool = (vis_frames // cfg.block_size - 1) * T
        cos, sin = wo.rope_tables(27, cfg.block_size, cfg.latent_height // 2, cfg.latent_width // 2)
        X = self.X
        t0 = time.perf_counter()
        m = p["mod"]
        xn = wo.layer_norm(X) * (1 + m[1]) + m[0]
        qkv = xn @ p["qkv_w"].T + p["qkv_b"]
        q = wo.apply_rope(wo.rms_norm(qkv[:, :d], p["nq"]).reshape(T, H, 128), cos, sin).reshape(T, d)
        k = wo.apply_rope(wo.rms_norm(qkv[:, d:2 * d], p["nk"]).reshape(T, H, 128), cos, sin).reshape(T, d)
        att = wo.attention(q, np.concatenate([self.pool_k[:npool], k]),
                           np.concatenate([self.pool_v[:npool], qkv[:, 2 * d:]]), H)
        Xo = X + m[2] * (att @ p["o_w"].T + p["o_b"])
        xc = wo.layer_norm(Xo) * p["n3w"] + p["n3b"]
        qc = wo.rms_norm(xc @ p["cq_w"].T + p["cq_b"], p["cnq"])
        Xo = Xo + wo.attention(qc, self.tk, self.tv, H) @ p["co_w"].T + p["co_b"]
        xm = wo.layer_norm(Xo) * (1 + m[4]) + m[3]
        Xo = Xo + m[5] * (wo.gelu_tanh(xm @ p["ffn1_w"].T + p["ffn1_b"]) @ p["ffn2_w"].T + p["ffn2_b"])
        return time.perf_counter() - t0


def trace_visible_frames(cfg):
    """Visible latent frames of every entry of the run, from the closed-form
    schedule and pool replay (oracle/schedule.py, restating the reference's
    tests/oracles.py:8-39): block k runs pass p at iteration k*o + p and
    enters the pool after its cache pass."""
    from oracle.schedule import enumerate_schedule, replay_pool, visible_blocks
    P, o, S = cfg.passes, cfg.offset, cfg.block_size
    rows = enumerate_schedule(cfg.num_blocks, P, o)
    out = []
    for i, row in enumerate(rows):
        inserted = [k for k in range(cfg.num_blocks) if k * o + P - 1 < i]
        pool, _ = replay_pool(inserted, cfg.window_blocks, cfg.sink_blocks)
        vis = visible_blocks([k for k, _ in row], pool, cfg.attention_mode)
        out += [len(v) * S for v in vis.values()]
    return out


def fit_line(points):
    """Least-squares t = a + b * frames over (frames, seconds) samples (per
    layer and entry, attention is linear in the visible keys, the rest is
    constant)."""
    xs = [float(x) for x, _ in points]
    ys = [float(y) for _, y in points]
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx if sxx > 0 else 0.0
    return my - b * mx, b


def cpu_run_seconds(cfg, points):
    """Host seconds of the whole run: layers x sum over the run's entries of
    the fitted per-layer time at that entry's visible-frame count."""
    a, b = fit_line(points)
    vis = trace_visible_frames(cfg)
    return cfg.layers * sum(a + b * v for v in vis), len(vis), (a, b)


def cpu_sample_frames(cfg):
    top = min(cfg.num_blocks, cfg.window_blocks + cfg.sink_blocks + cfg.cascade_width) * cfg.block_size
    return sorted({cfg.block_size, (cfg.block_size + top) // 2 // cfg.block_size * cfg.block_size, top})


def cpu_baseline(cfg, frames=None, pts=None):
    """cpu_baseline object for one config (rank 0, N=1): one timed layer
    sample at each of 2-3 distinct visible-frame counts, line fit, summed
    over the run's real entry list.  ``pts`` reuses another config's samples
    of the same model (same layer shapes; only the entry list differs)."""
    if pts is None:
        frames = frames or cpu_sample_frames(cfg)
        samp = CpuLayerSample(cfg, max(frames))
        samp.seconds(frames[0])                                # page-in
        pts = [(f, samp.seconds(f)) for f in frames]
    frames = [f for f, _ in pts]
    run_s, entries, (a, b) = cpu_run_seconds(cfg, pts)
    return {"value": cfg.num_blocks * FRAMES_PER_BLOCK / run_s, "unit": "frames/s",
            "cores": blas_threads(), "kind": "port",
            "sample": cpu_sample_desc(cfg, frames, entries),
            "sample_seconds": {str(f): round(t, 3) for f, t in pts},
            "fit_s_per_layer": [round(a, 4), round(b, 5)],
            "run_seconds_estimate": round(run_s, 1), "points": pts}


def cpu_sample_desc(cfg, frames, entries):
    return (f"numpy fp32 oracle (oracle/wan.py), BLAS threads {blas_threads()}: one layer of one entry "
            f"({cfg.tokens_per_block} query tokens, {cfg.text_len} text tokens) timed at visible frames "
            f"{frames}; t(frames) fitted linear and summed over the run's {entries} entries x "
            f"{cfg.layers} layers (embed/head/noise excluded)")


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


def parallelism(world):
    if world == 1:
        return "temporal1"
    from paper_2511_20426_b200.distributed import shard_mode
    how = os.environ.get("BC_KV_PUSH")
    push = ("copy-engine side stream" if how == "copy" else "q/k-kernel P2P stores" if how == "kernel" else
            "auto: copy engines between distinct GPUs, q/k-kernel P2P stores for ranks sharing a GPU")
    return f"temporal{world} (shard={shard_mode()}, kv_push={push}, IPC peer memory over NVLink)"


def workload_config(args, cfg, par):
    return {"workload": f"wan2.1-{args.preset} cascade o=1, {cfg.num_blocks} blocks "
                        f"({cfg.num_blocks * FRAMES_PER_BLOCK} frames), 480x832, 4-step, "
                        f"3 latent frames/block, {cfg.attention_mode}, W={cfg.window_blocks} "
                        f"sink={cfg.sink_blocks}"
                        + (f", cascade prompt switch every {args.switch_every} blocks"
                           if args.switch_every else ""),
            "model": f"wan2.1-{args.preset}-shaped", "global_batch": 1,
            "seq_len": cfg.tokens_per_block, "parallelism": par,
            "l2": "working set (weights + KV arena) >> 126 MB L2; no flush"}


def run_reference(args, cfg):
    """The reference arm: the oracle port of the path on the host cores.
    Each step times ONE layer of one entry at one visible-frame count
    (rotating over the counts the run has); value = the run's frames over
    the line fit summed across the run's real entry list x layers."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    vis = sorted(set(trace_visible_frames(cfg)))
    order = []
    lo, hi = 0, len(vis) - 1
    while lo <= hi:                       # extremes first: the fit is anchored early
        order.append(vis[hi])
        if lo != hi:
            order.append(vis[lo])
        lo, hi = lo + 1, hi - 1
    samp = CpuLayerSample(cfg, max(vis))
    for i in range(args.warmup):
        samp.seconds(order[i % len(order)])
    pts = [(order[i % len(order)], samp.seconds(order[i % len(order)])) for i in range(args.steps)]
    if len({f for f, _ in pts}) < 2:      # a line needs two distinct counts
        pts.append((order[1 % len(order)], samp.seconds(order[1 % len(order)])))
    run_s, entries, (a, b) = cpu_run_seconds(cfg, pts)
    fps = cfg.num_blocks * FRAMES_PER_BLOCK / run_s
    per = statistics.mean(t for _, t in pts)
    line = {
        "impl": "reference", "metric": metric_name(args),
        "value": fps, "unit": "frames/s", "n_gpus": max(world, args.gpus), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (random-init weights, N(0,1) activations)",
        "config": workload_config(args, cfg, "host cores (reference CPU path)"),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": blas_threads(), "kind": "port",
                         "sample": cpu_sample_desc(cfg, sorted({f for f, _ in pts}), entries),
                         "fit_s_per_layer": [a, b], "run_seconds_estimate": run_s},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

class Ctx:
    """Per-process measurement plumbing (ranks, barrier, max over ranks)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.world, self.rank, local = dist_env()
        # BC_FORCE_DEVICE / BC_DIST_BACKEND: test hooks to run the multi-rank
        # bench with several ranks on one GPU over gloo (NCCL refuses duplicate
        # GPUs); the driver's runs use one GPU per rank and NCCL
        self.dev = int(os.environ.get("BC_FORCE_DEVICE", local))
        self.backend = os.environ.get("BC_DIST_BACKEND", "nccl")
        torch.cuda.set_device(self.dev)
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group(self.backend)

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max(self, x):
        if self.world == 1:
            return x
        import torch.distributed as dist
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device="cuda" if self.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def device_timed(self, fn, steps, clocks_index=None):
        """K calls bracketed by barrier + synchronize, CUDA events on the
        launching stream; returns (max-over-ranks ms, results, clocks)."""
        torch = self.torch
        self.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(self.dev if clocks_index is None else clocks_index) as clocks:
            ev0.record()
            out = [fn() for _ in range(steps)]
            ev1.record()
            torch.cuda.synchronize()
        self.barrier()
        return self.max(ev0.elapsed_time(ev1)), out, clocks.summary()

    def host_timed(self, fn, steps):
        """End to end: host clock around K calls (host buffers in, results
        out), synchronize on both sides, max over ranks."""
        torch = self.torch
        self.barrier()
        torch.cuda.synchronize()
        with ClockSampler(self.dev) as clocks:
            t0 = time.perf_counter()
            out = [fn() for _ in range(steps)]
            torch.cuda.synchronize()
            s = time.perf_counter() - t0
        self.barrier()
        return self.max(s) * 1e3, out, clocks.summary()


def measure_config(C, bc, cfg, weights, steps, warmup, switches=(), seq=True, feed=None):
    """value (device-resident noise, graphs, no per-kernel events) and e2e
    (public run_cascade, host noise H2D, blocks D2H) for the cascade and, if
    asked, the sequential rollout of the same model -- both arms measured the
    same way (same K, W, clock and noise path)."""
    from paper_2511_20426_b200.metrics import streaming_fps
    from paper_2511_20426_b200.wan import ResidentNoiseFeed, run_noise_keys
    feed = feed or ResidentNoiseFeed(SESSION_SEED, cfg, run_noise_keys(cfg))
    frames = cfg.num_blocks * FRAMES_PER_BLOCK
    out = {}
    arms = [("cascade", cfg, bc.run_cascade)]
    if seq:
        arms.append(("sequential", bc.with_fields(cfg, offset=cfg.passes), None))
    for name, c, _ in arms:
        if name == "cascade":
            def dev_run(c=c):
                return bc.run_cascade(c, PROMPT, session_seed=SESSION_SEED, weights=weights,
                                      noise_feed=feed, switches=list(switches))

            def host_run(c=c):
                return bc.run_cascade(c, PROMPT, session_seed=SESSION_SEED, weights=weights,
                                      switches=list(switches))
        else:
            def dev_run(c=c):
                return bc.run_sequential_reference(c, PROMPT, session_seed=SESSION_SEED,
                                                   weights=weights, noise_feed=feed)

            def host_run(c=c):
                return bc.run_sequential_reference(c, PROMPT, session_seed=SESSION_SEED, weights=weights)
        for _ in range(warmup):
            dev_run()
        l0 = __import__("paper_2511_20426_b200._native", fromlist=["x"]).launch_count()
        ms, runs, clocks = C.device_timed(dev_run, steps)
        launches = __import__("paper_2511_20426_b200._native", fromlist=["x"]).launch_count() - l0
        host_run()                       # pinned staging / first-touch warm-up of the host path
        e2e_ms, _, clocks_e2e = C.host_timed(host_run, steps)
        out[name] = {"value": frames * steps / (ms / 1e3), "ms_per_step": ms / steps,
                     "streaming_fps": statistics.mean(streaming_fps(r.trace, clock="wall") for r in runs),
                     "e2e": frames * steps / (e2e_ms / 1e3), "e2e_ms_per_step": e2e_ms / steps,
                     "launches": launches, "clocks": clocks, "clocks_e2e": clocks_e2e,
                     "last_run": runs[-1]}
    return out, feed


def kernel_profile(bc, N, cfg, weights, feed):
    """Per-kernel-class breakdown in a SEPARATE pass: one generation launched
    eagerly with CUDA events around every launch on its stream
    (bc_profile_enable); the timed value above runs as CUDA graphs without
    events.  Returns ({class: (ms, flops, bytes, launches)}, run ms)."""
    import torch
    N.profile_collect()
    N.profile_enable(True)
    try:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bc.run_cascade(cfg, PROMPT, session_seed=SESSION_SEED, weights=weights, noise_feed=feed)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    finally:
        prof = N.profile_collect()
        N.profile_enable(False)
    return prof, wall


def kernel_times_graphs(bc, cfg, weights, feed, prof):
    """The same per-class breakdown in the PRODUCT launch mode: one generation
    launched as CUDA graphs without per-kernel events, kernel durations from
    CUPTI activity records (torch.profiler); algorithmic flops / bytes per
    class from the eager pass (they do not depend on the launch mode).
    Attention launches alternate self / cross within a layer (same kernel)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        bc.run_cascade(cfg, PROMPT, session_seed=SESSION_SEED, weights=weights, noise_feed=feed)
        torch.cuda.synchronize()
    evs = sorted((e for e in p.events() if e.device_type == torch.autograd.DeviceType.CUDA
                  and "bc::" in e.name), key=lambda e: e.time_range.start)
    out, k = {}, 0
    for e in evs:
        if "attn_sched_kernel" in e.name or "attn_kernel" in e.name:
            c = "self_attention" if k % 2 == 0 else "cross_attention"
            k += 1
        elif "gemm_kernel" in e.name:
            c = "gemm"
        else:
            c = "bandwidth"
        ms, n = out.get(c, (0.0, 0))
        out[c] = (ms + (e.time_range.end - e.time_range.start) / 1e3, n + 1)
    res = {}
    for c, (ms, n) in out.items():
        fl, by = (prof[c][1], prof[c][2]) if c in prof else (0.0, 0.0)
        res[c] = {"ms": round(ms, 3), "launches": n,
                  "tflops": round(fl / (ms / 1e3) / 1e12, 1) if fl > 0 and ms > 0 else None,
                  "gbs": round(by / (ms / 1e3) / 1e9, 1) if by > 0 and ms > 0 else None}
    return res


def kernels_and_roofline(prof, peaks, peak_kind):
    total = sum(v[0] for v in prof.values())
    kernels = {k: {"ms": round(v[0], 3), "launches": v[3],
                   "tflops": round(v[1] / (v[0] / 1e3) / 1e12, 1) if v[0] > 0 and v[1] > 0 else None,
                   "gbs": round(v[2] / (v[0] / 1e3) / 1e9, 1) if v[0] > 0 and v[2] > 0 else None,
                   "share": round(v[0] / total, 4) if total else None}
               for k, v in prof.items()}
    dom = max(("self_attention", "cross_attention", "gemm"), key=lambda k: prof[k][0])
    dom_ms, dom_flops, _, dom_n = prof[dom]
    achieved = dom_flops / (dom_ms / 1e3) / 1e12 if dom_ms > 0 else None
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get(dom)
    roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if achieved else None, "traffic": traffic,
            "peak_kind": f"{peak_kind} bf16 sustained", "launches": dom_n,
            "share_of_step": kernels[dom]["share"],
            "launch_mode": "separate profiled generation: eager launches, CUDA events around each "
                           "launch on its stream"}
    return kernels, roof


def sub_line(C, bc, name, cfg, weights, args, switches=(), seq=False, cpu_pts=None, feed=None,
             frames=None):
    """A secondary configuration (14B, LongLive-style, causal cascade): value
    and e2e measured like the headline with W = 1, K = 1 (a generation is
    2.4-20 s), plus its CPU baseline on rank 0 at N = 1 (same-model configs
    reuse the headline's layer samples, summed over their own entry list)."""
    steps = 1
    res, _ = measure_config(C, bc, cfg, weights, steps, 1, switches=switches, seq=seq, feed=feed)
    cas = res["cascade"]
    line = {"workload": name, "value": cas["value"], "unit": "frames/s", "steps": steps, "warmup": 1,
            "ms_per_step": cas["ms_per_step"], "streaming_fps": cas["streaming_fps"],
            "e2e": {"value": cas["e2e"], "unit": "frames/s"}, "gpu_launches": cas["launches"],
            "clocks": cas["clocks"]}
    if seq:
        s = res["sequential"]
        line["sequential"] = {"value": s["value"], "e2e": s["e2e"], "streaming_fps": s["streaming_fps"]}
    if C.world == 1 and C.rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, frames=frames, pts=cpu_pts)
    return line


def vae_report(C, bc, cfg, weights, feed, peaks):
    """VAE decode, timed separately as the north star asks:
    (a) the decoder alone on steady-state blocks (3 latent -> 12 video frames
    at 480x832), CUDA events on its stream; (b) the cascade and the sequential
    rollout with the decode lane on (each emitted block decoded on a side
    stream of the same GPU, overlapping the following iterations): frames
    over the time the LAST block finished decoding, and the paper's
    decode-inclusive streaming FPS."""
    import torch
    from paper_2511_20426_b200.metrics import end_to_end_fps, streaming_fps
    from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights, vae_config
    vcfg = vae_config("wan2.1", latent_h=cfg.latent_height, latent_w=cfg.latent_width,
                      block_size=cfg.block_size)
    dec = VaeDecoder(VaeWeights.random(vcfg, 11))
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    zs = [torch.randn((cfg.block_size, 16, cfg.latent_height, cfg.latent_width), generator=g, device="cuda")
          for _ in range(6)]
    dec.reset()
    dec.decode_block(zs[0])
    dec.decode_block(zs[1])
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(dec.stream)
    for z in zs[2:]:
        dec.decode_block(z)
    ev[1].record(dec.stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / (len(zs) - 2)
    fl = dec.flops_per_block(False)
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    out = {"decoder": "Wan2.1 causal 3-D VAE decoder (random init), 16 latent ch -> RGB, x8 space, x4 time",
           "ms_per_block": round(ms, 3), "video_frames_per_block": vcfg.frames_out(cfg.block_size, False),
           "decode_fps_alone": round(vcfg.frames_out(cfg.block_size, False) / ms * 1e3, 2),
           "tflop_per_block": round(fl / 1e12, 3), "tflops": round(fl / ms / 1e9, 1),
           "roofline_frac": round(fl / ms / 1e9 / peak, 4) if peak else None,
           "buffers_gb": round(dec.nbytes() / 1e9, 2)}
    for name, fn in (("cascade", bc.run_cascade), ("sequential", bc.run_sequential_reference)):
        c = cfg if name == "cascade" else bc.with_fields(cfg, offset=cfg.passes)
        fn(c, PROMPT, session_seed=SESSION_SEED, weights=weights, noise_feed=feed, decoder=dec)
        r = fn(c, PROMPT, session_seed=SESSION_SEED, weights=weights, noise_feed=feed, decoder=dec)
        out[f"{name}_with_decode"] = {
            "e2e_fps_decoded": round(end_to_end_fps(r.trace, clock="decoded"), 3),
            "streaming_fps_decoded": round(streaming_fps(r.trace, clock="decoded"), 3),
            "e2e_fps_generation_same_run": round(end_to_end_fps(r.trace), 3),
            "decode_lane": "same GPU, side stream, overlapped with the following iterations"}
    del dec
    torch.cuda.empty_cache()
    return out


def run_ours(args, cfg):
    import torch
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import _native as N
    from paper_2511_20426_b200.metrics import end_to_end_fps
    from paper_2511_20426_b200.wan import WanWeights, run_noise_keys

    C = Ctx()
    world, rank = C.world, C.rank
    weights = WanWeights.random(cfg, WEIGHT_SEED)
    switches = [bc.SwitchSpec(f"{PROMPT}, scene {k}", "cascade", at_block=k)
                for k in range(args.switch_every, cfg.num_blocks, args.switch_every)] \
        if args.switch_every else []
    frames = cfg.num_blocks * FRAMES_PER_BLOCK

    # ---- headline: cascade + sequential, value (resident noise, graphs,
    # no per-kernel events) and e2e (public API, host noise in, blocks out) ----
    res, feed = measure_config(C, bc, cfg, weights, args.steps, args.warmup, switches=switches,
                               seq=not args.no_seq)
    cas = res["cascade"]
    seq = res.get("sequential")

    # ---- per-kernel-class profile: separate eager pass ----
    prof, prof_ms = kernel_profile(bc, N, cfg, weights, feed)
    graphs = None
    if world == 1:
        try:
            graphs = kernel_times_graphs(bc, cfg, weights, feed, prof)
        except Exception as exc:   # the breakdown is informational; never lose the line
            graphs = {"error": f"{type(exc).__name__}: {exc}"[:200]}

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

    # ---- VAE decode, timed separately ----
    vae = None
    if world == 1 and not args.no_vae:
        vae = vae_report(C, bc, cfg, weights, feed, _peaks()[0])

    # ---- the reference's own CPU-runnable case (BASELINE configs[0]) ----
    toy = noise = cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        toy = toy_config1_times(bc)
        noise = noise_generation_report(cfg)
        cpu = cpu_baseline(cfg)

    # ---- secondary configurations (BASELINE configs[3], [4]; causal cascade) ----
    subs = {}
    if not args.no_sub and args.preset == "1.3b":
        subs["causal_cascade_1.3b"] = sub_line(
            C, bc, "wan2.1-1.3b cascade o=1, 13 blocks, CAUSAL attention among cascaded blocks",
            bc.with_fields(cfg, attention_mode="causal"), weights, args, seq=False,
            cpu_pts=cpu and cpu["points"])
        ll_cfg = bc.with_fields(cfg, total_frames=240, sink_blocks=0)
        ll_sw = [bc.SwitchSpec(f"{PROMPT}, scene {k}", "cascade", at_block=k) for k in (20, 40, 60)]
        subs["longlive_1.3b"] = sub_line(
            C, bc, "LongLive-style: wan2.1-1.3b cascade o=1, 80 blocks (240 latent / 960 video frames), "
                   "rolling W=7, no sink, cascade prompt switches at blocks 20/40/60, no KV recache",
            ll_cfg, weights, args, switches=ll_sw, seq=False, cpu_pts=cpu and cpu["points"])
        weights.runtime().release_cached()
        del weights
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        from paper_2511_20426_b200 import wan_config
        c14 = wan_config("14b", total_frames=cfg.total_frames, offset=1, attention_mode="bidirectional",
                         window_blocks=7, sink_blocks=cfg.sink_blocks)
        w14 = WanWeights.random(c14, WEIGHT_SEED)
        subs["wan14b"] = sub_line(
            C, bc, "wan2.1-14b-shaped cascade o=1, 13 blocks, 480x832, bidirectional, W=7 sink=1",
            c14, w14, args, seq=False, feed=feed, frames=[3, 39])
        w14.runtime().release_cached()
        del w14

    S = cfg.block_size
    lat_bytes = S * cfg.latent_dim * 4
    h2d = len(run_noise_keys(cfg)) * lat_bytes + cfg.text_len * cfg.text_dim * 4
    d2h = cfg.num_blocks * lat_bytes
    if rank != 0:
        return
    peaks, peak_kind = _peaks()
    kernels, roof = kernels_and_roofline(prof, peaks, peak_kind)
    line = {
        "metric": metric_name(args),
        "value": cas["value"], "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": cas["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": f"synthetic (random-init Wan2.1-{args.preset.upper()}-shaped weights, counter-keyed N(0,1) "
                "noise, hash-expanded 512x4096 text states)",
        "config": workload_config(args, cfg, parallelism(world)),
        "launch_mode": {"value": "CUDA graphs (one per batch width), no per-kernel events, noise "
                                 "pre-resident in HBM" if world == 1 else
                                 "eager multi-rank steps, noise pre-resident in HBM",
                        "e2e": "public run_cascade, host noise generated + copied H2D per iteration, "
                               "emitted blocks copied D2H, host clock",
                        "kernels": "separate eager generation with per-launch CUDA events",
                        "kernels_graphs": "one more generation as CUDA graphs (the product mode), kernel "
                                          "durations from CUPTI activity records (torch.profiler)"},
        "streaming_fps": cas["streaming_fps"],
        "sequential": ({"value": seq["value"], "e2e": seq["e2e"], "streaming_fps": seq["streaming_fps"],
                        "ms_per_step": seq["ms_per_step"], "steps": args.steps, "warmup": args.warmup,
                        "method": "same as the cascade: K timed generations after W warm-ups, device "
                                  "events with resident noise (value) and host clock with H2D noise (e2e)"}
                       if seq else None),
        "cascade_over_sequential": ({"value": cas["value"] / seq["value"], "e2e": cas["e2e"] / seq["e2e"],
                                     "streaming": cas["streaming_fps"] / seq["streaming_fps"]}
                                    if seq else None),
        "prompt_switch": switch,
        "vae_decode": vae,
        "config1_toy": toy,
        "noise_generation": noise,
        "roofline": roof,
        "kernels": kernels,
        "kernel_profile_run_ms": round(prof_ms, 1),
        "kernels_graphs": graphs,
        "e2e": {"value": cas["e2e"], "unit": "frames/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": cas["launches"],
        "clocks": cas["clocks"],
        "clocks_e2e": cas["clocks_e2e"],
        "cpu_baseline": cpu,
        "configs": subs or None,
    }
    print(json.dumps(line), flush=True)


def run_decode_gpu(args, cfg):
    """--decode-gpu (N >= 2 ranks): ranks 0..N-2 denoise (temporal
    parallelism over their own group), rank N-1 only runs the Wan2.1 VAE
    decoder; every emitted block goes rank 0 -> decode rank through the
    CUDA-IPC inbox (decode_rank.py).  A step
    = one generation AND the decode of all its blocks; value = video frames /
    max over ranks of (denoise time on the denoiser ranks, time of the last
    decode on the decode rank); generation-only and decode-inclusive
    streaming FPS reported beside it."""
    import torch
    import torch.distributed as dist
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import decode_rank as D
    from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights, vae_config
    from paper_2511_20426_b200.wan import ResidentNoiseFeed, WanWeights, run_noise_keys

    C = Ctx()
    if C.world < 2:
        raise SystemExit("--decode-gpu needs --gpus >= 2 (denoiser ranks + one decode rank)")
    is_dec, dec_rank = D.split_ranks(True)
    hand = D.DecodeHandoff(cfg, dec_rank)
    frames = cfg.num_blocks * FRAMES_PER_BLOCK
    if is_dec:
        vname = "tiny" if args.preset == "tiny" else "wan2.1"
        dec = VaeDecoder(VaeWeights.random(vae_config(vname, latent_h=cfg.latent_height,
                                                      latent_w=cfg.latent_width), 3))
        last = {}

        def run():
            last["times"] = hand.serve(dec, cfg.num_blocks)[1]
    else:
        weights = WanWeights.random(cfg, WEIGHT_SEED)
        feed = ResidentNoiseFeed(SESSION_SEED, cfg, run_noise_keys(cfg))
        remote = D.RemoteDecoder(hand)

        def run():
            return bc.run_cascade(cfg, PROMPT, session_seed=SESSION_SEED, weights=weights,
                                  noise_feed=feed, decoder=remote)
    for _ in range(args.warmup):
        run()
    C.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(C.dev) as clocks:
        ev0.record()
        for _ in range(args.steps):
            run()
        ev1.record()
        torch.cuda.synchronize()
    my_ms = ev0.elapsed_time(ev1)
    C.barrier()
    job_ms = C.max(my_ms)
    gen_ms = C.max(0.0 if is_dec else my_ms)
    dec_ms = C.max(my_ms if is_dec else 0.0)
    fps = C.max(D.decoded_fps(last["times"], FRAMES_PER_BLOCK)["streaming_fps_decoded"] if is_dec else 0.0)
    hand.close()
    if C.rank != 0:
        return
    G = C.world - 1
    line = {
        "metric": f"{metric_name(args)}, VAE-decoded on a separate GPU",
        "value": frames * args.steps / (job_ms / 1e3), "unit": "frames/s", "n_gpus": C.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": job_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init Wan2.1-shaped DiT and VAE decoder weights)",
        "config": workload_config(args, cfg, f"{parallelism(G)} + 1 decode GPU (rank {dec_rank})"),
        "generation_only": {"value": frames * args.steps / (gen_ms / 1e3), "ms_per_step": gen_ms / args.steps},
        "decode_rank": {"ms_per_step": dec_ms / args.steps, "streaming_fps_decoded": fps,
                        "handoff": "rank 0 -> decode rank: CUDA-IPC inbox ring (4 x 1.2 MB), "
                                   "peer copy + cuStreamWriteValue32 / cuStreamWaitValue32 flags"},
        "clocks": clocks.summary(),
    }
    if os.environ.get("BC_FORCE_DEVICE") is not None:
        line["note"] = ("all ranks time-share ONE GPU (BC_FORCE_DEVICE test hook): a functional run of "
                        "the multi-GPU path, not a performance number")
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args):
    """--gpus N>1 outside torchrun: one process per GPU under
    torch.distributed.run (127.0.0.1 rendezvous); rank 0 prints the line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--preset", default="1.3b")
    ap.add_argument("--blocks", type=int, default=13)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline samples")
    ap.add_argument("--sink", type=int, default=1, help="sink blocks (LongLive-style: 0)")
    ap.add_argument("--switch-every", type=int, default=0,
                    help="cascade-mode prompt switch every N blocks")
    ap.add_argument("--no-seq", action="store_true", help="skip the sequential rollout")
    ap.add_argument("--no-vae", action="store_true", help="skip the VAE decode measurements")
    ap.add_argument("--no-switch", action="store_true",
                    help="skip the cascade-vs-recache prompt-switch measurement")
    ap.add_argument("--no-sub", action="store_true",
                    help="skip the 14B / LongLive / causal secondary configurations")
    ap.add_argument("--decode-gpu", action="store_true",
                    help="N >= 2: the last rank only VAE-decodes (SURVEY 8f rank 1), fed by rank 0")
    args = ap.parse_args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    from paper_2511_20426_b200 import wan_config
    cfg = wan_config(args.preset, total_frames=3 * args.blocks, offset=1,
                     attention_mode="bidirectional", window_blocks=7, sink_blocks=args.sink)
    if args.impl == "reference":
        run_reference(args, cfg)
    elif args.decode_gpu:
        run_decode_gpu(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
