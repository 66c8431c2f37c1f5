"""The real one-process-per-rank path (DistWanSession: CUDA-IPC-mapped peer
KV replicas, P2P K/V stores, ready flags, stream-memop Y waits, done epochs, output
gather) with two processes sharing cuda:0 over a gloo group.  The GPU
time-slices the two contexts; outputs must equal the single-process run
bit-for-bit (placement independence, reference test_acceptance.py:58-76)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q, mode, shard):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      BC_TEMPORAL_SHARD=shard.split("+")[0],
                      BC_NOISE_GATHER="1" if shard.endswith("+gather") else "0")
    if shard.endswith("+kflags"):   # peer flags published by the kernel fallback, not stream memops
        os.environ["BC_NO_MEMOP_WRITES"] = "1"
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_20426_b200 as bc
        from paper_2511_20426_b200.wan import WanWeights
        cfg = bc.wan_config("tiny", total_frames=15, attention_mode=mode)
        w = WanWeights.random(cfg, 7)
        run = bc.run_cascade(cfg, "a lighthouse in a storm", weights=w)
        if rank == 0:
            q.put({b: run.outputs[b] for b in run.outputs})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,shard", [("bidirectional", "rows"), ("causal", "rows"),
                                        ("bidirectional", "blocks"), ("bidirectional", "rows+gather"),
                                        ("bidirectional", "rows+kflags")])
def test_two_processes_one_gpu(mode, shard):
    """rows+gather: the host noise draws are split over the ranks and
    all-gathered (the NCCL path, here over gloo through the host)."""
    import torch.multiprocessing as mp
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200.wan import WanWeights
    from conftest import rel_l2, wan_oracle_outputs
    cfg = bc.wan_config("tiny", total_frames=15, attention_mode=mode)
    w = WanWeights.random(cfg, 7)
    base = bc.run_cascade(cfg, "a lighthouse in a storm", weights=w)
    ref = wan_oracle_outputs(cfg, w, "a lighthouse in a storm")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, mode, shard)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(got) == sorted(base.outputs)
    for b in base.outputs:
        assert np.array_equal(got[b], base.outputs[b]), b
        assert rel_l2(got[b], ref[b]) < 1e-2, b   # and the two-rank run vs the fp32 oracle
