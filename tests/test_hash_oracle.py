"""CPU: the hash oracle (oracle/hash_fold64.c + fold64_py) against the
reference's frozen vectors and reference-generated golden digests."""
import json
import os

import pytest

from oracle import hash_ref

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hash_vectors.json")))


def test_ts_cross_language_vectors():
    for hexp, want in GOLD["ts_vectors"]:
        p = bytes.fromhex(hexp)
        assert hash_ref.fold64_py(p) == int(want)
        assert hash_ref.fold64_c(p) == int(want)


def test_stability_vector():
    p = eval(GOLD["stability"]["expr"])  # bytes(range(256)) * 4096
    assert hash_ref.fold64_c(p) == int(GOLD["stability"]["digest"]) == 3578566749703741650


def test_every_length_1_to_4096():
    bl = GOLD["by_length"]
    for n in range(1, 4097):
        p = hash_ref.payload(n, bl["seed"], n)
        assert hash_ref.fold64_c(p) == int(bl["digests"][n - 1]), n
    for n in (1, 7, 8, 9, 63, 64, 65, 255):
        assert hash_ref.fold64_py(hash_ref.payload(n, bl["seed"], n)) == int(bl["digests"][n - 1])


def test_large_payloads():
    for item in GOLD["large"]:
        p = hash_ref.payload(item["len"], item["seed"], item["content_id"])
        assert hash_ref.fold64_c(p) == int(item["digest"])


def test_batch_mt_matches_single():
    import numpy as np
    bufs = [hash_ref.payload(n, 3, n) for n in (1, 9, 100, 4096, 70000)]
    arrs = [np.frombuffer(b, dtype=np.uint8) for b in bufs]
    ptrs = np.array([a.ctypes.data for a in arrs], dtype=np.uint64)
    lens = np.array([a.size for a in arrs], dtype=np.uint64)
    one = hash_ref.fold64_c_batch(ptrs, lens, threads=1)
    mt = hash_ref.fold64_c_batch(ptrs, lens, threads=3)
    assert list(one) == list(mt) == [hash_ref.fold64_py(b) for b in bufs]


def test_oracle_matches_reference_live():
    from tests.conftest import import_reference
    dmlens = import_reference()
    import random
    rng = random.Random(5)
    for _ in range(300):
        p = rng.randbytes(rng.randint(1, 300))
        assert hash_ref.fold64_c(p) == dmlens.hash_bytes(p)


def test_empty_rejected():
    with pytest.raises(ValueError):
        hash_ref.fold64_py(b"")
