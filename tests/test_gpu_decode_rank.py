"""VAE decode on a dedicated GPU: the last
rank of the job only decodes, the others denoise in their own process group,
and every emitted block travels rank 0 -> decode rank through the CUDA-IPC
inbox ring with stream-memory-operation flags (decode_rank.py).  Here the
processes share cuda:0 over a gloo world group (the protocol never spins on
an SM, so time-sliced ranks cannot starve each other).  The decoded videos
must equal a single-process run with the decoder on the same GPU bit for
bit, and the denoiser outputs must equal the single-process run."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PROMPT = "a lighthouse in a storm"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfgs():
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200.vae import vae_config
    cfg = bc.wan_config("tiny", total_frames=27)
    vcfg = vae_config("tiny", latent_h=cfg.latent_height, latent_w=cfg.latent_width)
    return cfg, vcfg


def _rank(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), BC_TEMPORAL_SHARD="rows")
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_20426_b200 as bc
        from paper_2511_20426_b200 import decode_rank as D
        from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights
        from paper_2511_20426_b200.wan import WanWeights
        cfg, vcfg = _cfgs()
        is_dec, dec_rank = D.split_ranks(True)
        hand = D.DecodeHandoff(cfg, dec_rank)
        if is_dec:
            dec = VaeDecoder(VaeWeights.random(vcfg, 3))
            dist.barrier()
            videos, times = hand.serve(dec, cfg.num_blocks)
            q.put(("videos", {b: v.cpu().numpy() for b, v in videos.items()}, times))
        else:
            w = WanWeights.random(cfg, 7)
            dist.barrier()
            run = bc.run_cascade(cfg, PROMPT, weights=w, decoder=D.RemoteDecoder(hand))
            if rank == 0:
                q.put(("outputs", {b: run.outputs[b] for b in run.outputs}, None))
        hand.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_decode_on_a_dedicated_rank(world):
    """world 2: one denoiser rank (single-GPU session) + the decode rank;
    world 3: two denoiser ranks (rows partition, their own group) + decode."""
    import torch
    import torch.multiprocessing as mp
    import paper_2511_20426_b200 as bc
    from paper_2511_20426_b200 import decode_rank as D
    from paper_2511_20426_b200.vae import VaeDecoder, VaeWeights
    from paper_2511_20426_b200.wan import WanWeights
    cfg, vcfg = _cfgs()
    base = bc.run_cascade(cfg, PROMPT, weights=WanWeights.random(cfg, 7),
                          decoder=VaeDecoder(VaeWeights.random(vcfg, 3)))
    want = {b: v.cpu().numpy() for b, v in base.videos.items()}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((kind, (payload, times)) for kind, payload, times in (q.get(timeout=600), q.get(timeout=600)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    outs, _ = got["outputs"]
    assert sorted(outs) == sorted(base.outputs)
    for b in base.outputs:
        assert np.array_equal(outs[b], base.outputs[b]), b
    videos, times = got["videos"]
    assert sorted(videos) == list(range(cfg.num_blocks))
    for b in range(cfg.num_blocks):
        assert np.array_equal(videos[b], want[b]), b
    done = [t[1] for t in times]
    assert all(t1 >= t0 >= 0.0 for t0, t1 in times) and done == sorted(done)
    fps = D.decoded_fps(times, cfg.block_size * cfg.video_frames_per_latent)
    assert fps["e2e_fps_decoded"] > 0.0 and fps["streaming_fps_decoded"] > 0.0
    del torch
