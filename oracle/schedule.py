"""Closed-form schedule and pool oracles -- TEST ORACLE ONLY.

Restates /root/reference/pkg/tests/oracles.py:8-39 (enumerate_schedule,
replay_pool) and the build_mask visibility rule (denoiser.py:172-194).
"""

from __future__ import annotations


def enumerate_schedule(num_blocks, passes, offset):
    """Block k runs pass p at iteration k*offset + p (oracles.py:8-21)."""
    total = (num_blocks - 1) * offset + passes
    return [[(k, t - k * offset) for k in range(num_blocks) if 0 <= t - k * offset < passes]
            for t in range(total)]


def replay_pool(inserts, window, sink_blocks):
    """Keep every inserted block, then drop the smallest non-sink indices
    while more than ``window`` are held (oracles.py:24-39)."""
    held, evicted = [], []
    for b in inserts:
        if b not in held:
            held.append(b)
        held.sort()
        regular = [x for x in held if not (sink_blocks and x == 0)]
        while len(regular) > window:
            v = regular.pop(0)
            held.remove(v)
            evicted.append(v)
    return held, evicted


def visible_blocks(batch, pool, mode):
    """Per query block: ascending visible key blocks (denoiser.py:172-194)."""
    keys = sorted(pool) + sorted(batch)
    return {q: sorted(k for k in keys if mode == "bidirectional" or k <= q)
            for q in sorted(batch)}
