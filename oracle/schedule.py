"""Closed-form schedule and pool oracles -- TEST ORACLE ONLY.

Restates /root/reference/pkg/tests/oracles.py:8-39 (enumerate_schedule,
replay_pool) and the build_mask visibility rule (denoiser.py:172-194).
"""

from __future__ import annotations


def enumerate_schedule(num_blocks, passes, offset):
    """Block k runs pass p at iteration k*offset + p (oracles.py:8-21):
    brute force over every (block, pass) pair, bucketed by iteration."""
    rows = [[] for _ in range((num_blocks - 1) * offset + passes)]
    for k in range(num_blocks):
        for p in range(passes):
            rows[k * offset + p].append((k, p))
    return rows


def replay_pool(inserts, window, sink_blocks):
    """Hold every inserted block; while more than ``window`` non-sink blocks
    are held, evict the smallest (oracles.py:24-39).  Returns (held, evicted)."""
    held, evicted = set(), []
    for b in inserts:
        held.add(b)
        pinned = {0} & held if sink_blocks else set()
        regular = sorted(held - pinned)
        drop = regular[:max(0, len(regular) - window)]
        held.difference_update(drop)
        evicted.extend(drop)
    return sorted(held), evicted


def visible_blocks(batch, pool, mode):
    """Per query block: ascending visible key blocks (denoiser.py:172-194)."""
    keys = sorted(pool) + sorted(batch)
    return {q: sorted(k for k in keys if mode == "bidirectional" or k <= q)
            for q in sorted(batch)}
