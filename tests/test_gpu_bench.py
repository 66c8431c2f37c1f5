"""bench.py on the GPU: `--gpus 2` outside torchrun re-launches itself as
two ranks (here both on cuda:0 over gloo through the BC_FORCE_DEVICE /
BC_DIST_BACKEND test hooks; the driver's runs use one GPU per rank over
NCCL) and prints ONE line with n_gpus = 2."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("gpus", [1, 2])
def test_bench_line(gpus):
    env = dict(os.environ, BC_FORCE_DEVICE="0", BC_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                          "--preset", "tiny", "--blocks", "9", "--steps", "2", "--warmup", "1",
                          "--no-cpu", "--no-sub", "--no-switch"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and d["roofline"]["achieved"] > 0
    assert d["sequential"]["value"] > 0
    if gpus > 1:
        assert "shard=" in d["config"]["parallelism"]
    else:
        v = d["vae_decode"]
        assert v["ms_per_block"] > 0 and v["cascade_with_decode"]["e2e_fps_decoded"] > 0
        g = d["kernels_graphs"]      # product launch mode, CUPTI kernel durations
        assert g["self_attention"]["ms"] > 0 and g["gemm"]["launches"] == d["kernels"]["gemm"]["launches"]


@pytest.mark.parametrize("gpus", [2, 3])
def test_bench_decode_gpu_line(gpus):
    """--decode-gpu: the last rank only VAE-decodes, fed by rank 0 through the
    IPC inbox; one line, value over the whole job."""
    env = dict(os.environ, BC_FORCE_DEVICE="0", BC_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--decode-gpu",
                          "--preset", "tiny", "--blocks", "9", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["value"] > 0 and d["generation_only"]["value"] >= d["value"] * 0.999
    assert "decode GPU" in d["config"]["parallelism"] and d["decode_rank"]["streaming_fps_decoded"] > 0
