"""Host-side logic: config, scheduler, pool, masks, metrics, switches
(reference tests test_config/test_core/test_scheduler/test_kvpool/
test_metrics/test_interactive restated against this package)."""

import math
import random

import numpy as np
import pytest

import paper_2511_20426_b200 as bc
from oracle.schedule import enumerate_schedule, replay_pool


def drive(num_blocks, offset, workers=1):
    st = bc.CascadeState(num_blocks=num_blocks, offset=offset,
                         schedule=bc.make_schedule([1000, 750, 500, 250]), workers=workers)
    plans = []
    while not st.done:
        p = bc.plan_iteration(st)
        plans.append(p)
        bc.advance(st, p, p.blocks)
    return st, plans


def test_schedule_examples():
    s = bc.make_schedule([1000, 750, 500, 250])
    assert (s.passes, s.emit_pass, s.cache_pass) == (5, 3, 4)
    assert s.table() == [1000, 750, 500, 250, 0.0]
    for bad in ([], [1200], [1000, 0], [500, 500], [float("nan")], [500, 750]):
        with pytest.raises(bc.InvalidInputError):
            bc.make_schedule(bad)


def test_steady_state_plan_and_counts():
    _, plans = drive(13, 1)
    assert [(e.block_index, e.noise_level) for e in plans[9].entries] == \
        [(5, 0.0), (6, 250.0), (7, 500.0), (8, 750.0), (9, 1000.0)]
    for o in range(1, 6):
        for b in range(1, 25):
            _, plans = drive(b, o)
            assert len(plans) == (b - 1) * o + 5
            assert [[(e.block_index, e.pass_index) for e in p.entries] for p in plans] == \
                enumerate_schedule(b, 5, o)


def test_phases_and_snapshot_resume():
    st = bc.CascadeState(num_blocks=13, offset=1, schedule=bc.make_schedule([1000, 750, 500, 250]))
    seen = []
    for _ in range(9):
        seen.append(st.phase)
        p = bc.plan_iteration(st)
        bc.advance(st, p)
    assert seen[0] == "fill" and "steady" in seen
    clone = bc.CascadeState.from_snapshot(st.to_snapshot())
    while not st.done:
        a, b = bc.plan_iteration(st), bc.plan_iteration(clone)
        assert a == b
        bc.advance(st, a)
        bc.advance(clone, b)
    assert clone.done and clone.phase == "done"
    with pytest.raises(bc.ContractViolation):
        bc.plan_iteration(st)


def test_pool_eviction_against_replay_oracle():
    rng = random.Random(7)
    for _ in range(300):
        window, sink = rng.randint(1, 6), rng.choice([0, 1])
        inserts = [rng.randint(0, 15) for _ in range(rng.randint(0, 25))]
        pool = bc.KVPool.empty(window, sink)
        for b in inserts:
            pool = pool.insert(b, (bc.LayerKV(b, 0, np.zeros((3, 1, 1)), np.zeros((3, 1, 1)), 0.0, "c"),))
        assert pool.block_indices == replay_pool(inserts, window, sink)[0]


def test_pool_evicted_by_and_mismatch():
    kv = lambda b: (bc.LayerKV(b, 0, np.zeros((3, 1, 1)), np.zeros((3, 1, 1)), 0.0, "c"),)
    pool = bc.KVPool.empty(2, 1)
    for b in range(3):
        pool = pool.insert(b, kv(b))
    newer = pool.insert(3, kv(3))
    assert pool.evicted_by(newer) == [1] and newer.block_indices == [0, 2, 3]
    with pytest.raises(bc.ContractViolation):
        pool.insert(2, kv(3))


def test_slot_allocator_reuse():
    from paper_2511_20426_b200.kvpool import SlotAllocator
    a = SlotAllocator(3)
    s0, s1 = a.acquire(10), a.acquire(11)
    assert a.acquire(10) == s0 and s0 != s1
    a.release(10)
    assert a.acquire(12) == s0
    a.acquire(13)
    with pytest.raises(bc.ContractViolation):
        a.acquire(14)


def test_config_rules_and_wan_presets(tmp_path):
    assert bc.CascadeConfig().validate().cascade_width == 5
    with pytest.raises(bc.InvalidInputError):
        bc.CascadeConfig(window_blocks=2, sink_blocks=1, offset=1).validate()
    with pytest.raises(bc.InvalidInputError) as err:
        bc.CascadeConfig(block_size=0, workers=-1).validate()
    assert {"block_size", "workers"} <= set(err.value.fields)
    c = bc.wan_config("1.3b")
    assert (c.model_dim, c.tokens_per_block, c.latent_dim, c.num_blocks) == (1536, 4680, 99840, 13)
    c14 = bc.wan_config("14b")
    assert (c14.model_dim, c14.layers, c14.ffn_dim) == (5120, 40, 13824)
    with pytest.raises(bc.InvalidInputError):
        bc.with_fields(c, latent_dim=16)
    path = tmp_path / "cfg.yaml"
    bc.dump_config(c, path)
    assert bc.load_config(path) == c
    env = {"CASCADE_OFFSET": "2", "CASCADE_ATTENTION_MODE": "causal"}
    assert bc.load_config(path, environ=env).offset == 2
    with pytest.raises(bc.InvalidInputError):
        bc.load_config(overrides={"nonsense": 1})


def test_mask_lists_are_prefixes_in_engine_shapes():
    from paper_2511_20426_b200.denoiser import visible_block_lists
    m = bc.build_mask([5, 6, 7], [0, 2, 3, 4], "causal", 3)
    assert visible_block_lists(m) == [[0, 2, 3, 4, 5], [0, 2, 3, 4, 5, 6], [0, 2, 3, 4, 5, 6, 7]]
    m = bc.build_mask([5, 6], [4], "bidirectional", 3)
    assert m.visible_frames(5) == 9


def test_metrics_definitions():
    tr = bc.Trace()
    clock = 0.0
    for i in range(13):
        step = {7: 0.5, 8: 0.375}.get(i, 1.0)
        frames = {7: 14}.get(i, 12)
        clock += step
        tr.append(bc.TraceEvent(iteration=i, entries=[], wall_seconds=step, modeled_exec=1.0,
                                modeled_comm=0.0, modeled_stall=0.0, modeled_decode=0.0,
                                modeled_clock=clock, wall_clock=clock, pool_blocks=0, pool_frames=0,
                                pool_state=[], emitted_block=i, emitted_video_frames=frames))
    assert bc.streaming_fps(tr) == 30.0
    assert bc.streaming_fps(tr, clock="wall") == 30.0
    assert math.isclose(bc.end_to_end_fps(tr), (12 * 12 + 14) / clock)
    with pytest.raises(bc.ContractViolation):
        tr.append(tr.events[0])


def test_switch_spec_and_queue():
    s = bc.SwitchSpec("x", "cascade", at_block=8)
    assert s.boundary_iteration(1, 3) == 11
    with pytest.raises(bc.InvalidInputError):
        bc.SwitchSpec("x", "cascade")
    q = bc.CommandQueue()
    r = q.submit(bc.LiveSwitchRequest("p"))
    assert q.pop() is r and q.pop() is None
    q.submit(r)
    q.reject_all(bc.InvalidInputError("done"))
    with pytest.raises(bc.InvalidInputError):
        r.wait(0.1)


def test_engine_recache_accounting(oracle_engine, default_config):
    """A recache switch pays one pass per pool block (stall on the modeled
    clock, pool re-tagged level 0 / new prompt); a cascade switch pays none."""
    cfg = bc.with_fields(default_config, total_frames=24)
    run = bc.run_cascade(cfg, "p", switches=[bc.SwitchSpec("q", "recache", at_block=6)])
    ev = run.switch_events[0]
    hit = next(e for e in run.trace.events if e.switch is not None)
    assert ev.extra_passes == hit.pool_blocks and hit.modeled_stall == ev.stall_modeled > 0
    assert all(row["noise_tag"] == 0.0 and row["conditioning_id"] == ev.conditioning_id
               for row in hit.pool_state)
    plain = bc.run_cascade(cfg, "p", switches=[bc.SwitchSpec("q", "cascade", at_block=6)])
    assert plain.switch_events[0].extra_passes == 0
    assert run.trace.events[-1].modeled_clock == plain.trace.events[-1].modeled_clock + ev.stall_modeled


def test_engine_properties_on_oracle(oracle_engine, default_config):
    """Reference acceptance properties through the product engine (CPU oracle forward)."""
    cfg = bc.with_fields(default_config, total_frames=18)
    base = bc.run_cascade(cfg, "determinism")
    multi = bc.run_cascade(bc.with_fields(cfg, workers=5), "determinism")
    for k in base.outputs:
        assert np.array_equal(base.outputs[k], multi.outputs[k])
    seq = bc.run_sequential_reference(cfg, "p")
    cas = bc.run_cascade(bc.with_fields(cfg, offset=5), "p")
    for k in seq.outputs:
        assert np.array_equal(seq.outputs[k], cas.outputs[k])
    assert bc.attention_cost(bc.run_cascade(bc.with_fields(cfg, total_frames=3), "p").trace) == 45
    bc.verify_schedule_consistency(base.trace, cfg)


def test_trace_export_import_round_trip(oracle_engine, default_config, tmp_path):
    """json-lines export is lossless (reference metrics.py:181-205); the CSV
    carries the instantaneous-FPS series; bad formats and clocks raise."""
    from paper_2511_20426_b200.metrics import export_trace, import_trace
    run = bc.run_cascade(bc.with_fields(default_config, total_frames=18), "p")
    export_trace(run.trace, tmp_path / "t.jsonl")
    back = import_trace(tmp_path / "t.jsonl")
    assert [e.to_json() for e in back.events] == [e.to_json() for e in run.trace.events]
    assert back.total_passes == run.trace.total_passes == 30
    export_trace(run.trace, tmp_path / "t.csv", format="csv")
    rows = (tmp_path / "t.csv").read_text().splitlines()
    series = bc.instantaneous_fps(run.trace)
    assert rows[0] == "block_index,video_frames,elapsed,fps" and len(rows) == 1 + len(series) == 7
    assert rows[1].split(",")[0] == str(series[0].block_index) and float(rows[1].split(",")[3]) == series[0].fps
    assert series.fps_values() == [p.fps for p in series.points]
    with pytest.raises(bc.InvalidInputError):
        export_trace(run.trace, tmp_path / "t.x", format="xml")
    with pytest.raises(bc.InvalidInputError):
        bc.instantaneous_fps(run.trace, clock="cpu")
    with pytest.raises(bc.InvalidInputError):
        bc.streaming_fps(run.trace)  # 6 blocks < 9


def test_row_slices_partition_properties():
    """rows partition: contiguous, disjoint, covering slices of the n*T rows,
    balanced to one unit, cut only at query-tile boundaries of an entry, and
    producer masks consistent with the slices."""
    from paper_2511_20426_b200.distributed import ROW_TILE, entry_producers, row_slices
    for n in range(1, 6):
        for T in (48, 192, 300, 4680):
            for g in range(1, 9):
                sl = row_slices(n, T, g)
                assert len(sl) == g
                nonempty = [s for s in sl if s[1] > s[0]]
                assert nonempty[0][0] == 0 and nonempty[-1][1] == n * T
                for (a0, a1), (b0, b1) in zip(nonempty, nonempty[1:]):
                    assert a1 == b0
                unit = ROW_TILE if n * -(-T // ROW_TILE) >= 2 * g else 16
                for a, b in sl:
                    for x in (a, b):
                        assert x == n * T or (x % T) % unit == 0     # tile boundary inside its entry
                tiles = [len(range(0, T, unit)) * n]
                counts = []
                for a, b in sl:
                    c = sum(1 for e in range(n) for t in range(0, T, unit) if a <= e * T + t < b)
                    counts.append(c)
                assert sum(counts) == tiles[0] and max(counts) - min(counts) <= 1
                masks = entry_producers(sl, n, T)
                for e, m in enumerate(masks):
                    owners = {r for r, (a, b) in enumerate(sl) if a < (e + 1) * T and b > e * T}
                    assert m == sum(1 << r for r in owners) and m


def test_modeled_clock_acceptance_properties(oracle_engine):
    """Reference acceptance (test_acceptance.py:79-99) through the product
    engine's modeled clock: B = 40, o = 1, G = 5, uniform pass cost, zero
    comm/decode -> modeled speedup exactly 200/44 over the sequential
    rollout; positive comm or decode cost strictly lowers it; the streaming
    FPS ratio of the 13-block paper config vs sequential is exactly 5."""
    paper = bc.CascadeConfig(total_frames=39, block_size=3, latent_dim=16, window_blocks=7,
                             sink_blocks=1, offset=1, workers=1, pass_cost_base=1.0).validate()
    prompt = "a lighthouse in a storm"
    cfg = bc.with_fields(paper, total_frames=120, workers=5)

    def speedup(c):
        seq = bc.run_sequential_reference(c, prompt).trace.total_modeled_time
        return seq / bc.run_cascade(c, prompt).trace.total_modeled_time

    ideal = 200.0 / 44.0
    s = speedup(cfg)
    assert abs(s - ideal) <= 1e-9 and s < 5.0
    assert speedup(bc.with_fields(cfg, comm_cost_per_frame=1e-4)) < ideal
    assert speedup(bc.with_fields(cfg, decode_cost=1e-2)) < ideal
    cascade = bc.run_cascade(bc.with_fields(paper, workers=5), prompt)
    sequential = bc.run_sequential_reference(paper, prompt)
    assert bc.streaming_fps(cascade.trace) / bc.streaming_fps(sequential.trace) == 5.0


def _attention_plan(vis, q_tokens, kv_tokens, heads):
    import ctypes as C
    from paper_2511_20426_b200 import _native as N
    b = N.make_batch(3, list(range(len(vis))), [0.0] * len(vis), [0] * len(vis), vis)
    items = np.zeros(6144, np.uint32)
    start = np.zeros(257, np.uint16)
    n_ctas = C.c_int32()
    n = N.lib().bc_attention_plan(C.byref(b), q_tokens, kv_tokens, heads, items.ctypes.data, 6144,
                                  start.ctypes.data, C.byref(n_ctas))
    assert n >= 0
    return items[:n], start[:n_ctas.value + 1]


@pytest.mark.parametrize("vis,q_tokens,heads", [
    ([list(range(13))] * 5, 4680, 12),                    # steady state, bidirectional
    ([[0, 1, 2], [0, 1, 2, 3], [0, 1, 2, 3, 4]], 4680, 12),  # causal-like: no equal lists
    ([[0, 1], [2, 3], [0, 1], [2, 3], [0, 1]], 328, 12),     # two groups of equal lists
    ([[0, 1]] * 2, 4680, 40),                              # 14B head count
    ([list(range(13))] * 5, 4680, 40),                    # 14B steady state (must not fall back)
    ([[0]], 300, 2),                                       # fewer items than CTAs
])
def test_attention_work_list_covers_every_tile_once(vis, q_tokens, heads):
    """The balanced attention kernel's work list (built on the host,
    csrc/attention.cu build_sched): every (entry, head, 128-row query tile)
    appears in exactly one item; pairs are consecutive tiles of one entry;
    cross-entry pairs join the last tiles of two entries with identical
    visible lists; the CTAs' modelled loads differ by at most one item."""
    items, start = _attention_plan(vis, q_tokens, 256, heads)
    nq = -(-q_tokens // 128)
    seen = {}
    load = []
    for c in range(len(start) - 1):
        cost = 0.0
        for w in items[start[c]:start[c + 1]]:
            w = int(w)
            e, h = w & 0xff, (w >> 8) & 0xff
            if w & 0x40000000:
                e2 = (w >> 16) & 0xff
                assert e2 != e and vis[e] == vis[e2]
                tiles = [(e, h, nq - 1), (e2, h, nq - 1)]
                cost += 2 * len(vis[e])
            elif w & 0x80000000:
                t = (w >> 16) & 0x3fff
                assert t + 1 < nq
                tiles = [(e, h, t), (e, h, t + 1)]
                cost += 2 * len(vis[e])
            else:
                tiles = [(e, h, (w >> 16) & 0x3fff)]
                cost += 1.8 * len(vis[e])
            for k in tiles:
                assert k not in seen, k
                seen[k] = True
        load.append(cost)
    assert len(seen) == len(vis) * heads * nq
    biggest = 2 * max(len(v) for v in vis)
    assert max(load) - min(load) <= biggest + 1e-9


def test_attention_plan_rejects_malformed_batches():
    """bc_attention_plan is a public entry point: visible counts beyond
    BC_MAX_VIS, bad head / token counts are contract errors, not stack
    overwrites."""
    import ctypes as C
    from paper_2511_20426_b200 import _native as N
    b = N.make_batch(3, [0], [0.0], [0], [[0]])
    items = np.zeros(64, np.uint32)
    start = np.zeros(257, np.uint16)
    n_ctas = C.c_int32()
    b.n_vis[0] = 10_000
    assert N.lib().bc_attention_plan(C.byref(b), 128, 256, 2, items.ctypes.data, 64, start.ctypes.data,
                                     C.byref(n_ctas)) == 1
    b.n_vis[0] = 1
    for q, kv, h in ((0, 256, 2), (128, 0, 2), (128, 256, 0), (128, 256, 256)):
        assert N.lib().bc_attention_plan(C.byref(b), q, kv, h, items.ctypes.data, 64, start.ctypes.data,
                                         C.byref(n_ctas)) == 1


class _FakeCtx:
    """Stands in for wan._Ctx in the operator-arena bookkeeping tests (no GPU)."""

    def __init__(self, n_slots, layers=2):
        self.n_slots, self.layers, self.handle = n_slots, layers, object()
        self.reads = []

    def read_kv(self, slot, layer, which):
        self.reads.append((slot, layer, which))
        return np.zeros((3, 1, 1))


def test_operator_arena_slots_generations_and_residency():
    """Wan operator path (wan.WanRuntime.forward): a fresh block takes the
    least recently used slot the call does not attend to; recycling a slot
    bumps its generation so the old handle raises instead of reading another
    block's K/V; handles come back resident whether passed as the SlotKV or
    as the reference KVPool's tuple of its layers (kvpool.py:51-53)."""
    from paper_2511_20426_b200.errors import ContractViolation
    from paper_2511_20426_b200.kvpool import SlotKV
    from paper_2511_20426_b200.wan import _OpArena
    op = _OpArena(_FakeCtx(4))
    s0 = op.take(set(), 0)
    h0 = SlotKV(op.ref(s0), s0, 0, 0.0, "c", 3)
    assert op.resident_slot(h0) == s0 and op.resident_slot(tuple(h0)) == s0
    pinned = {s0}
    s1 = op.take(pinned, 1)
    assert s1 != s0
    h1 = SlotKV(op.ref(s1), s1, 1, 0.0, "c", 3)
    # a call attending to block 0 never hands its slot to a new block
    for b in range(2, 12):
        s = op.take({s0}, b)
        assert s != s0
    assert op.resident_slot(h0) == s0 and h0[1].keys.shape == (3, 1, 1)
    # block 1's slot was recycled meanwhile: its handle is stale
    assert op.resident_slot(h1) is None
    with pytest.raises(ContractViolation):
        h1[0].keys
    # a tuple mixing layers of different handles is not a resident block
    assert op.resident_slot((h0[0], h1[1])) is None
    with pytest.raises(ContractViolation):
        op.take({0, 1, 2, 3}, 99)


def test_decoded_fps_definitions():
    """decode_rank.decoded_fps: end to end = all frames / last decode done;
    streaming = mean of 12 frames over the intervals ending at blocks 8 and 9
    (1-indexed) on the decode rank's clock."""
    from paper_2511_20426_b200.decode_rank import decoded_fps
    times = [(0.1 * b, 0.1 * b + 0.05) for b in range(13)]
    times[8] = (0.8, 0.95)         # block 9 (1-indexed) finishes late
    f = decoded_fps(times, 12)
    assert f["e2e_fps_decoded"] == pytest.approx(13 * 12 / 1.25)
    assert f["streaming_fps_decoded"] == pytest.approx((12 / 0.1 + 12 / 0.2) / 2)
    assert decoded_fps(times[:5], 12)["streaming_fps_decoded"] is None


@pytest.mark.parametrize("M,N,K,mode,want", [
    (23400, 4608, 1536, 0, (256, 2)),   # QKV at width 5
    (23400, 1536, 1536, 3, (192, 2)),   # o / cross-o (gated residual) at width 5
    (23400, 8960, 1536, 1, (256, 2)),   # FFN1 (GELU)
    (23400, 1536, 8960, 3, (192, 2)),   # FFN2 (gated residual)
    (4680, 1536, 1536, 3, (224, 2)),    # width-1 o / cross-o: 2 waves of 224-wide pairs (3 of 128 x 1: +8%)
    (18720, 1536, 1536, 3, (192, 2)),   # width 4: 8 exact waves of 192, not 7 of ragged 224
    (4680, 1536, 8960, 3, (224, 2)),    # width-1 FFN2: 7 column tiles of 224 (last one ragged)
    (4680, 1536, 1536, 0, (224, 2)),    # width-1 cross-attention q projection
    (4680, 4608, 1536, 0, (256, 2)),    # width-1 QKV: 5 waves of 256 beat 6 of 224
    (2925, 1536, 8960, 3, (256, 2)),    # a G = 8 row slice: one wave of pairs
])
def test_gemm_tiling_choices(M, N, K, mode, want):
    """The cost-model tiling (gemm.cu gemm_plan) picks the tilings measured
    fastest for the DiT's shapes (scripts/gemm_tiling.py,
    profiles/r2_gemm_tiling.txt); host logic, no GPU needed."""
    import ctypes
    from paper_2511_20426_b200 import _native as nat
    bn, cg = ctypes.c_int32(), ctypes.c_int32()
    nat.check(nat.lib().bc_gemm_plan(M, N, K, mode, ctypes.byref(bn), ctypes.byref(cg)), "bc_gemm_plan")
    assert (bn.value, cg.value) == want
    assert (N % bn.value == 0 or bn.value == 224) and (bn.value not in (192, 224) or cg.value == 2)


def test_attention_sequential_shape_one_pair_one_lone_tile():
    """The width-1 (sequential rollout) self-attention launch: 12 heads x 37
    query tiles = 444 tiles on 148 CTAs -- the balanced work list gives every
    CTA one ping-pong pair and one lone tile (the lone
    tile's exposed softmax is where the sequential rollout loses ~20% of its
    attention time; splitting its key range would break P1 bit-exactness)."""
    import collections
    items, start = _attention_plan([list(range(8))], 4680, 256, 12)
    kinds = collections.Counter()
    for c in range(len(start) - 1):
        k = sorted("P" if int(w) & 0x80000000 else "X" if int(w) & 0x40000000 else "S"
                   for w in items[start[c]:start[c + 1]])
        kinds["".join(k)] += 1
    assert len(start) - 1 == 148 and kinds == {"PS": 148}
