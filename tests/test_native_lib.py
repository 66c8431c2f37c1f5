"""The C-ABI library loads on a CPU-only machine and exports every entry
point include/bcb200.h declares; host-side (non-GPU) entry points work."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "bcb200.h")).read()
    return sorted(set(re.findall(r"\b(bc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2511_20426_b200 import _native
    handle = ctypes.CDLL(_native.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 15
    missing = [s for s in declared if not hasattr(handle, s)]
    assert not missing, missing
    assert sorted(_native.exported_symbols()) == declared
    assert b"sm_100a" in _native.lib().bc_version()


def test_philox_words_match_numpy():
    from paper_2511_20426_b200 import _native
    for key, ctr in [((7, 0), (0, 0, 0, 0)), ((2 ** 64 - 1, 12345), (2 ** 64 - 2, 5, 9, 1))]:
        bg = np.random.Philox(key=np.array(key, dtype=np.uint64),
                              counter=np.array(ctr, dtype=np.uint64))
        want = bg.random_raw(4)          # numpy increments the counter before the block
        inc = list(ctr)
        for i in range(4):
            inc[i] = (inc[i] + 1) % 2 ** 64
            if inc[i] != 0:
                break
        assert _native.philox4x64(key, inc) == [int(x) for x in want]


@pytest.mark.parametrize("seed,ctr,n", [(20260809, (0, 0, 0, 0), 1), (3, (1, 2, 3, 0), 99840),
                                        (2 ** 63 + 5, (2 ** 64 - 1, 2 ** 64 - 1, 1, 0), 4097)])
def test_native_noise_bit_exact(seed, ctr, n):
    from paper_2511_20426_b200 import _native
    want = np.random.Generator(np.random.Philox(key=np.uint64(seed),
                                                counter=np.array(ctr, dtype=np.uint64))).standard_normal(n)
    out64 = np.empty(n)
    out32 = np.empty(n, dtype=np.float32)
    _native.run_noise_tasks([(seed, 0, ctr, out64)], 0)
    _native.run_noise_tasks([(seed, 0, ctr, out32)], 1)
    assert np.array_equal(out64, want)
    assert np.array_equal(out32, want.astype(np.float32))


def test_block_noise_threads_order_independent():
    from paper_2511_20426_b200 import NoiseStream
    ns = NoiseStream(99, 4096)
    a = ns.block_noise(3, 2, 9, 3)
    b = np.stack([ns.draw(3, 2, 9 + i) for i in range(3)])
    assert np.array_equal(a, b)


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2511_20426_b200 as bc
    with pytest.raises(bc.DeviceError):
        bc.renoise(np.zeros((3, 4)), np.zeros((3, 4)), 10.0)
    w = bc.init_model(1, 1, 1, 4, 4)
    with pytest.raises(bc.DeviceError):
        bc.forward(w, [bc.EntryInput(0, np.zeros((3, 4)), 1000.0, bc.embed_prompt("x", 4))], [],
                   bc.build_mask([0], [], "causal", 3))
