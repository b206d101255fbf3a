"""Small invocations of every analysis kernel path for compute-sanitizer (memcheck / racecheck /
synccheck): C2 and C4 traces (the C4 hash palette drives the fix-up's long-run fallback), the
stable-sort strategies on adversarial keys, and the device-resident sharded pipeline."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_12713_b200 import _lib, analyze_columns, savings_columns, sharded  # noqa: E402
from paper_2601_12713_b200.synth import c2_trace, c4_trace  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
for c in (c2_trace(n), c4_trace(n)):
    cf = analyze_columns(c)
    sv = savings_columns(c, cf)
    cs = analyze_columns(c, strict=True)
    print("ok", cf.counts(), cs.counts())
L = _lib.lib()
L.b2l_stable_sort_u64.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p]
rng = np.random.default_rng(5)
top = rng.integers(0, 2**63, 16, dtype=np.uint64) & np.uint64(0xFFFFFF0000000000)
keys = np.concatenate([t | (rng.integers(0, 4, 40, dtype=np.uint64) * np.uint64(0x10001)) for t in top])
keys = np.concatenate([keys, rng.choice(rng.integers(0, 2**63, 64, dtype=np.uint64), 3000)])
for strategy in (0, 1, 16 + 5):
    perm = np.zeros(keys.size, np.uint32)
    _lib.check(L.b2l_stable_sort_u64(keys.ctypes.data, keys.size, strategy, perm.ctypes.data), "sort")
    assert np.array_equal(perm, np.argsort(keys, kind="stable")), strategy
print("ok sorts")
if "--no-sharded" in sys.argv:  # (racecheck on the threaded sharded run alone takes > 10 min)
    sys.exit(0)
c = c2_trace(n)
got = sharded.run_local_device(c, 2)
assert got.counts() == analyze_columns(c).counts()
print("ok sharded", got.counts())
