"""bench.py's reference arm (the driver runs `bench.py --impl reference`):
one JSON line with the contract keys, on a tiny preset so it runs on CPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--preset", "tiny", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]


def test_noise_generation_report_tiny():
    """The bench's separate host-noise report: native generator
    draws for every (block, pass) key of a run, checked against numpy."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2511_20426_b200 as bc
    cfg = bc.wan_config("tiny", total_frames=9)
    r = bench.noise_generation_report(cfg)
    assert r["bit_identical_to_numpy"] and r["block_passes_per_run"] == 3 * 4
    assert r["bytes_per_run"] == 12 * cfg.block_size * cfg.latent_dim * 4 and r["native_ms_per_run"] > 0


def test_trace_visible_frames_matches_engine_trace(oracle_engine):
    """The CPU arm sums its fitted per-layer time over the run's entries;
    the entry list (visible frames per entry, from the closed-form schedule
    and pool replay) equals what the product engine's trace records."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2511_20426_b200 as bc
    for kw in (dict(offset=1), dict(offset=5), dict(offset=2, attention_mode="causal"),
               dict(offset=1, sink_blocks=0, window_blocks=5)):
        cfg = bc.CascadeConfig(total_frames=39, pass_cost_base=1.0, **kw).validate()
        run = bc.run_cascade(cfg, "a red cube")
        want = [e["visible_frames"] for ev in run.trace.events for e in ev.entries]
        assert bench.trace_visible_frames(cfg) == want, kw


def test_fit_line_exact():
    sys.path.insert(0, ROOT)
    import bench
    a, b = bench.fit_line([(3, 1.0 + 0.5 * 3), (21, 1.0 + 0.5 * 21), (39, 1.0 + 0.5 * 39)])
    assert abs(a - 1.0) < 1e-12 and abs(b - 0.5) < 1e-12
