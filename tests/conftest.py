import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(os.path.join(GOLDEN, "toy_golden.npz"), allow_pickle=False))


@pytest.fixture(scope="session")
def golden_sched():
    import json
    with open(os.path.join(GOLDEN, "schedule_golden.json")) as fh:
        return json.load(fh)


TINY = dict(layers=4, latent_dim=256, heads=2, head_dim=128, cond_dim=256,
            total_frames=18, offset=1, window_blocks=7, sink_blocks=1,
            attention_mode="bidirectional", pass_cost_base=1.0)


@pytest.fixture(scope="session")
def tiny_config():
    from paper_2511_20426_b200 import CascadeConfig
    return CascadeConfig(**TINY).validate()


@pytest.fixture(scope="session")
def default_config():
    from paper_2511_20426_b200 import CascadeConfig
    return CascadeConfig(total_frames=39, pass_cost_base=1.0).validate()


@pytest.fixture
def oracle_engine(monkeypatch):
    """Route the product engine's device runtime to the CPU oracle session
    (test seam; the product never does this)."""
    from paper_2511_20426_b200 import engine
    from oracle.loop import oracle_runtime
    monkeypatch.setattr(engine, "_runtime_for", oracle_runtime)
    return engine


def wan_oracle_outputs(cfg, weights, prompt, device_oracle=False, switches=()):
    """Outputs of the product engine driven by the Wan oracle (numpy fp32 on
    the host, or its torch fp32 restatement on the GPU for big geometry)
    instead of the device runtime -- the checker for multi-rank runs."""
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import engine
    from oracle.loop import wan_oracle_runtime, wan_torch_oracle_runtime
    rt = wan_torch_oracle_runtime(weights.t) if device_oracle else wan_oracle_runtime(weights.host_params())
    orig = engine._runtime_for
    engine._runtime_for = rt
    try:
        run = bc.run_cascade(bc.with_fields(cfg, workers=1), prompt, weights=weights, switches=list(switches))
    finally:
        engine._runtime_for = orig
    return run.outputs


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
