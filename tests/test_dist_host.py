"""Host-side logic of the multi-GPU path with world_size 2 over gloo on CPU:
every rank derives the same slot tables and wait epochs from the shared
schedule, and the ranks' entry sets partition every plan."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_20426_b200 as bc
        from paper_2511_20426_b200.distributed import (SlotEpochs, entry_producers, need_table,
                                                       rank_entries, row_slices)
        from paper_2511_20426_b200.kvpool import SlotAllocator
        from paper_2511_20426_b200.denoiser import visible_block_lists
        cfg = bc.wan_config("tiny", total_frames=39, workers=world)
        T = cfg.tokens_per_block
        logs = {}
        for mode in ("blocks", "rows"):
            st = bc.CascadeState(num_blocks=cfg.num_blocks, offset=cfg.offset, schedule=cfg.schedule())
            pool = bc.KVPool.empty(cfg.window_blocks, cfg.sink_blocks)
            n_slots = cfg.window_blocks + cfg.sink_blocks + cfg.cascade_width + 1
            slots, epochs = SlotAllocator(n_slots), SlotEpochs(n_slots)
            log = []
            while not st.done:
                plan = bc.plan_iteration(st)
                epoch = plan.iteration + 1
                for b in plan.blocks:
                    slots.acquire(b)
                mask = bc.build_mask(plan.blocks, pool.block_indices, "bidirectional", cfg.block_size)
                vis = visible_block_lists(mask)
                n = len(plan.blocks)
                if mode == "rows":
                    sl = row_slices(n, T, world)
                    masks = entry_producers(sl, n, T)
                    local, prod = list(range(n)), dict(zip(plan.blocks, masks))
                else:
                    sl, prod = None, None
                    local = rank_entries(plan.blocks, world, rank)
                    masks = [1 << (b % world) for b in plan.blocks]
                need, pm = need_table([plan.blocks[i] for i in local], [vis[i] for i in local],
                                      plan.blocks, epochs, epoch, world, rank, slots.slot_of, prod)
                log.append({"local": [plan.blocks[i] for i in local], "need": need, "pmask": pm,
                            "slots": [slots.slot_of(b) for b in plan.blocks], "slices": sl,
                            "vis": [vis[i] for i in local], "masks": masks})
                epochs.wrote([slots.slot_of(b) for b in plan.blocks], epoch, masks)
                bc.advance(st, plan)
                for e in plan.entries:
                    if e.pass_index == cfg.schedule().cache_pass:
                        kv = (bc.LayerKV(e.block_index, 0, None, None, 0.0, "c"),)
                        newer = pool.insert(e.block_index, kv)
                        for gone in pool.evicted_by(newer):
                            slots.release(gone)
                        pool = newer
            logs[mode] = log
        everyone = [None] * world
        dist.all_gather_object(everyone, logs)
        if rank == 0:
            q.put(everyone)
    finally:
        dist.destroy_process_group()


def test_two_rank_host_agreement():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    logs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # blocks partition: owner = block % world; a peer-owned visible block is waited for
    a, b = logs[0]["blocks"], logs[1]["blocks"]
    assert len(a) == len(b) == 17
    for it, (ra, rb) in enumerate(zip(a, b)):
        assert ra["slots"] == rb["slots"]                       # same slot table on every rank
        assert sorted(ra["local"] + rb["local"]) == sorted(set(ra["local"] + rb["local"]))
        assert all(x % 2 == 0 for x in ra["local"]) and all(x % 2 == 1 for x in rb["local"])
        for r, log in ((0, ra), (1, rb)):
            for blk_vis, row, mrow in zip(log["vis"], log["need"], log["pmask"]):
                for vb, need, m in zip(blk_vis, row, mrow):
                    if vb % 2 == r:
                        assert need == 0 and m == 0               # own writes are stream-ordered
                    else:
                        assert 1 <= need <= it + 1 and m == 1 << (vb % 2)  # a peer published it
    # rows partition: every rank runs every entry on a disjoint row slice
    a, b = logs[0]["rows"], logs[1]["rows"]
    for it, (ra, rb) in enumerate(zip(a, b)):
        assert ra["slots"] == rb["slots"] and ra["slices"] == rb["slices"]
        assert ra["local"] == rb["local"] and len(ra["local"]) == len(ra["slots"])
        (a0, a1), (b0, b1) = ra["slices"]
        assert a0 == 0 and a0 < a1 == b0 < b1 == len(ra["slots"]) * 192   # tiny: T = 192 tokens
        for r, log in ((0, ra), (1, rb)):
            for row, mrow in zip(log["need"], log["pmask"]):
                for need, m in zip(row, mrow):
                    assert not (m >> r) & 1                       # never wait on yourself
                    assert (need == 0) == (m == 0) and need <= it + 1


def _split_worker(rank, world, port, q, shard):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), BC_TEMPORAL_SHARD=shard)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_20426_b200 import decode_rank, distributed
        from paper_2511_20426_b200.errors import InvalidInputError
        try:
            is_dec, dec = decode_rank.split_ranks(True)
        except InvalidInputError:
            q.put((rank, "rejected"))
            return
        # the denoiser group holds ranks 0..N-2; the decode rank is outside it
        n = dist.get_world_size(distributed.DIT_GROUP) if not is_dec else None
        q.put((rank, (is_dec, dec, n, distributed.dit_world() if not is_dec else None)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shard", ["rows", "blocks"])
def test_decode_rank_split_three_ranks(shard):
    """decode_rank.split_ranks over gloo, world 3: ranks 0-1 denoise in their
    own group, rank 2 decodes; the blocks partition is rejected on EVERY rank
    before any collective (a decode GPU needs every block on rank 0)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, 3, port, q, shard)) for r in range(3)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if shard == "blocks":
        assert got == {0: "rejected", 1: "rejected", 2: "rejected"}
    else:
        assert got == {0: (False, 2, 2, 2), 1: (False, 2, 2, 2), 2: (True, 2, None, None)}
