"""Hash oracle (TEST INFRASTRUCTURE ONLY).

* ``fold64_py``   -- pure-Python restatement of dmlens.hashing._fold64 +
  make_hasher (/root/reference/pkg/src/dmlens/hashing.py:34-64), for small cases.
* ``fold64_c`` / ``fold64_c_batch`` -- the same algorithm in plain C
  (oracle/hash_fold64.c, built into oracle/liborc_hash.so by oracle/Makefile).

Pinned against the reference's 12 frozen cross-language vectors
(pkg/shim/test/hash64.test.ts:8-24), the 1 MiB stability vector
(pkg/tests/test_hashing.py:62-74) and digests produced by the reference's own
hash_bytes (tests/golden/hash_vectors.json, made by tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "liborc_hash.so")
M64 = (1 << 64) - 1


def fold64_py(payload: bytes) -> int:
    n = len(payload)
    if n == 0:
        raise ValueError("cannot hash a zero-byte payload")
    h = 0xCBF29CE484222325
    padded = payload + b"\0" * (-n % 8)
    for i in range(0, len(padded), 8):
        h = ((h ^ int.from_bytes(padded[i:i + 8], "little")) * 0x100000001B3) & M64
    h ^= n
    for mult in (0xFF51AFD7ED558CCD, 0xC4CEB9FE1A85EC53):
        h ^= h >> 33
        h = (h * mult) & M64
    h ^= h >> 33
    return h or 1


_lib = None


def build() -> str:
    src = os.path.join(_HERE, "hash_fold64.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        L.orc_hash_bytes.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.orc_hash_bytes.restype = ctypes.c_uint64
        L.orc_hash_batch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        L.orc_hash_batch_mt.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                        ctypes.c_int]
        L.orc_hash_batch_mt.restype = ctypes.c_int
        L.orc_payload_word.argtypes = [ctypes.c_uint64] * 3
        L.orc_payload_word.restype = ctypes.c_uint64
        L.orc_fill_payload.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        _lib = L
    return _lib


def fold64_c(payload) -> int:
    arr = np.frombuffer(bytes(payload), dtype=np.uint8)
    if arr.size == 0:
        raise ValueError("cannot hash a zero-byte payload")
    return int(lib().orc_hash_bytes(arr.ctypes.data, arr.size))


def fold64_c_batch(ptrs: np.ndarray, lens: np.ndarray, threads: int = 1) -> np.ndarray:
    """Digests of host buffers given as uint64 address / length arrays."""
    out = np.zeros(len(ptrs), dtype=np.uint64)
    if threads <= 1:
        lib().orc_hash_batch(ptrs.ctypes.data, lens.ctypes.data, len(ptrs), out.ctypes.data)
    else:
        rc = lib().orc_hash_batch_mt(ptrs.ctypes.data, lens.ctypes.data, len(ptrs), out.ctypes.data, threads)
        if rc != 0:
            raise RuntimeError("orc_hash_batch_mt failed")
    return out


def payload(nbytes: int, seed: int, content_id: int) -> bytes:
    """Synthetic payload bytes (same stream as the device generator b2l_fill_payloads)."""
    buf = np.zeros(nbytes, dtype=np.uint8)
    if nbytes:
        lib().orc_fill_payload(buf.ctypes.data, nbytes, seed, content_id)
    return buf.tobytes()


def audit_ref(observations):
    """Restatement of dmlens.hashing.CollisionAuditStore.observe (hashing.py:70-87) over
    (hash, payload) observations in order -> (collision_count, distinct hashes)."""
    first, count = {}, 0
    for h, p in observations:
        if h not in first:
            first[h] = bytes(p)
        elif first[h] != p:
            count += 1
    return count, len(first)
