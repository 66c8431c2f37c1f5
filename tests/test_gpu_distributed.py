"""Multi-GPU temporal-parallel device path, exercised on ONE GPU by
EmulatedRanks: G rank contexts with their own KV-arena replicas, P2P pushes
into each other's arenas, (layer, slot) ready flags and iteration-done
flags -- the same kernels and host logic as one-process-per-GPU.  Outputs
must be bit-identical to the single-rank run for every G (reference
test_acceptance.py:58-76 worker determinism), and every replica must hold
the same pool KV."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200.wan import WanWeights
    cfg = bc.wan_config("tiny", total_frames=18)
    return cfg, WanWeights.random(cfg, 7)


def _stack(run):
    return np.stack([run.outputs[k] for k in sorted(run.outputs)])


@pytest.mark.parametrize("mode,push", [("bidirectional", "copy"), ("causal", "copy"),
                                       ("bidirectional", "kernel")])
def test_emulated_ranks_bit_identical(tiny, monkeypatch, mode, push):
    """push = copy: copy engines + stream memory ops move the fresh K/V and
    publish the flags; push = kernel: P2P stores from the q/k kernel."""
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import distributed
    monkeypatch.setenv("BC_KV_PUSH", push)
    cfg, w = tiny
    cfg = bc.with_fields(cfg, attention_mode=mode)
    base = bc.run_cascade(cfg, "a lighthouse in a storm", weights=w)
    monkeypatch.setattr(distributed, "EMULATE", True)
    for g in (2, 3, 5, 8):
        run = bc.run_cascade(bc.with_fields(cfg, workers=g), "a lighthouse in a storm", weights=w)
        assert np.array_equal(_stack(run), _stack(base)), g
        assert run.pool.state_dump() == base.pool.state_dump()


def test_emulated_replicas_agree(tiny, monkeypatch):
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import distributed, engine
    cfg, w = tiny
    monkeypatch.setattr(distributed, "EMULATE", True)
    captured = {}
    orig_close = distributed.EmulatedRanks.close

    def close(self):
        torch.cuda.synchronize()
        captured["arenas"] = [a.clone() for a in self.replica_arenas()]
        captured["slots"] = dict(self.slots.owner)
        orig_close(self)

    monkeypatch.setattr(distributed.EmulatedRanks, "close", close)
    run = bc.run_cascade(bc.with_fields(cfg, workers=3), "p", weights=w)
    arenas, slots = captured["arenas"], captured["slots"]
    for b in run.pool.block_indices:
        s = slots[b]
        for a in arenas[1:]:
            assert torch.equal(a[:, s], arenas[0][:, s]), b


def test_emulated_prompt_switch(tiny, monkeypatch):
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import distributed
    cfg, w = tiny
    sw = [bc.SwitchSpec("second scene", "cascade", at_block=2)]
    base = bc.run_cascade(cfg, "first", weights=w, switches=sw)
    monkeypatch.setattr(distributed, "EMULATE", True)
    run = bc.run_cascade(bc.with_fields(cfg, workers=2), "first", weights=w, switches=sw)
    assert np.array_equal(_stack(run), _stack(base))
