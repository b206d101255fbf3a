"""Generates the committed golden fixtures from the UNMODIFIED reference.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py
The fixtures travel with the repo; nothing at test time reads /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("DMLENS_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from dmlens.hashing import hash_bytes  # noqa: E402  (the reference's own implementation)

from oracle.hash_ref import payload  # noqa: E402  (deterministic payload bytes only)

# frozen cross-language vectors of the reference (pkg/shim/test/hash64.test.ts:8-24)
TS_VECTORS = [
    ("00", 13822439871872589623), ("ff", 12844647536454529852), ("61", 2714998891557577425),
    ("616263", 16769191619139763278), ("6162636465666768", 2402220733500462054),
    ("616263646566676869", 11245955420054164285),
    ("000102030405060708090a0b0c0d0e0f", 13029654848220864353),
    ("aa" * 7, 17947520978646933045), ("55" * 63, 4886044645629322746),
    (bytes(range(256)).hex(), 5613354006569079831),
    (bytes(i % 251 for i in range(1024)).hex(), 11562279238887807506),
    ("00" * 32, 9077827906869418884),
]


def hash_fixture():
    out = {"ts_vectors": [], "stability": None, "by_length": {}, "large": []}
    for hexp, want in TS_VECTORS:
        got = hash_bytes(bytes.fromhex(hexp))
        assert got == want, (hexp, got, want)
        out["ts_vectors"].append([hexp, str(want)])
    stab = bytes(range(256)) * 4096
    out["stability"] = {"expr": "bytes(range(256)) * 4096", "digest": str(hash_bytes(stab))}
    seed = 7
    out["by_length"] = {"seed": seed, "content_id": "length", "lengths": "1..4096",
                        "digests": [str(hash_bytes(payload(n, seed, n))) for n in range(1, 4097)]}
    for i, n in enumerate([1024, 4097, 65536, 131077, 262144, 1048576, 1048573]):
        out["large"].append({"len": n, "seed": 11, "content_id": 1000 + i,
                             "digest": str(hash_bytes(payload(n, 11, 1000 + i)))})
    return out


if __name__ == "__main__":
    with open(os.path.join(HERE, "hash_vectors.json"), "w") as f:
        json.dump(hash_fixture(), f, indent=0)
    print("wrote hash_vectors.json")
