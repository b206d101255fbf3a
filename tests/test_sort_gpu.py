"""GPU stable-sort strategies behind the grouping steps (detectors.py:85-191 group by content
hash, device and address; groups are then ordered by first start): plain LSD, the wide
prefix + segmented fix-up sort, and prefix sorts at every split byte.  Each must equal a
stable CPU argsort on adversarial keys: long equal runs, prefix collisions between distinct
keys, runs straddling the fix-up limit and tile edges."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIX_T = 32  # run limit of the in-place fix-up (b2l_prims.cuh)


def _sort(keys, strategy):
    from paper_2601_12713_b200 import _lib
    L = _lib.lib()
    L.b2l_stable_sort_u64.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p]
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    perm = np.zeros(keys.size, dtype=np.uint32)
    _lib.check(L.b2l_stable_sort_u64(keys.ctypes.data, keys.size, strategy, perm.ctypes.data),
               "b2l_stable_sort_u64")
    return perm


def _cases():
    rng = np.random.default_rng(2601)
    full = lambda m: rng.integers(0, 2**63, m, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, m, dtype=np.uint64)
    out = {
        "random": full(300_000),
        "palette_64k": rng.choice(full(65_536), 400_000),  # C4-style hash palette: long runs
        "all_equal": np.full(10_000, 0xDEADBEEF12345678, np.uint64),
        "sorted": np.sort(full(50_000)),
        "reverse": np.sort(full(50_000))[::-1].copy(),
        "one_byte": rng.integers(0, 256, 70_000, dtype=np.uint64) << np.uint64(40),
        "tiny": full(3),
    }
    # distinct keys sharing the top 3 bytes, interleaved, runs around the fix-up limit
    top = full(64) & np.uint64(0xFFFFFF0000000000)
    parts = []
    for j, t in enumerate(top):
        m = [FIX_T - 1, FIX_T, FIX_T + 1, 2 * FIX_T + 3][j % 4]
        low = rng.integers(0, 4, m, dtype=np.uint64) * np.uint64(0x10001)
        parts.append(t | low)
    coll = np.concatenate(parts)
    out["prefix_collisions"] = rng.permutation(coll)
    out["prefix_runs_in_order"] = coll
    for m in (2047, 2048, 2049, 4095, 4097):  # tile edges of the fix-up and onesweep
        out[f"edge_{m}"] = rng.choice(full(m // 3 + 1), m)
    return out


@pytest.mark.parametrize("strategy", [0, 1] + [16 + b for b in range(8)])
def test_stable_sort_strategies_match_numpy(cuda, strategy):
    for name, keys in _cases().items():
        want = np.argsort(keys, kind="stable").astype(np.uint32)
        got = _sort(keys, strategy)
        assert np.array_equal(got, want), (name, strategy)


def test_wide_sort_large_random(cuda):
    rng = np.random.default_rng(7)
    keys = rng.integers(0, 2**63, 4_000_000, dtype=np.uint64)
    keys[::5] = keys[1::5]  # 20% duplicated hashes
    assert np.array_equal(_sort(keys, 1), np.argsort(keys, kind="stable").astype(np.uint32))
