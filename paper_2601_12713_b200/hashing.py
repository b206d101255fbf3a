"""Content hashing on the B200 -- drop-in for dmlens.hashing.

Same contract as the reference (pkg/src/dmlens/hashing.py:22-67): FNV-1a-64
over little-endian u64 words with a zero-extended tail word, ``^= len``,
murmur3 fmix64, a computed 0 remapped to 1, and ``EmptyPayload`` for a
zero-byte payload.  Every digest is computed by the sm_100a kernel
``k_hash_seq`` in libb2l.so; there is no CPU path.

Entry points
  hash_bytes(payload) -> int                 HashFn drop-in (hashing.py:67)
  make_hasher(raw) -> HashFn                 contract wrapper (hashing.py:55-64)
  hash_batch(payloads) -> list[int]          many host buffers, one pipelined call
  hash_tensors(tensors) -> torch.Tensor      device-resident buffers (no copies)
  hash_device(ptrs, lens, out, order, stream) raw device batch (C ABI b2l_hash_batch)
"""
from __future__ import annotations

import ctypes
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from .errors import EmptyPayload

HashFn = Callable[[bytes], int]
U64_MASK = (1 << 64) - 1


def _host_view(payload):
    """(address, length, keepalive) of a bytes-like host buffer without copying when possible."""
    if isinstance(payload, bytes):
        return ctypes.cast(ctypes.c_char_p(payload), ctypes.c_void_p).value, len(payload), payload
    if isinstance(payload, np.ndarray):
        arr = np.ascontiguousarray(payload)
        return arr.ctypes.data, arr.nbytes, arr
    mv = memoryview(payload)
    if not mv.contiguous:
        data = mv.tobytes()
        return ctypes.cast(ctypes.c_char_p(data), ctypes.c_void_p).value, len(data), data
    arr = np.frombuffer(mv.cast("B"), dtype=np.uint8) if mv.nbytes else np.zeros(0, np.uint8)
    return (arr.ctypes.data if arr.size else 0), mv.nbytes, arr


def _fold64_device(payload) -> int:
    addr, n, keep = _host_view(payload)
    if n == 0:
        raise EmptyPayload()
    out = ctypes.c_uint64(0)
    _lib.check(_lib.lib().b2l_hash_bytes(addr, n, ctypes.byref(out)), "b2l_hash_bytes")
    del keep
    return out.value


def make_hasher(raw: Callable[[bytes], int]) -> HashFn:
    """Producer contract wrapper, as dmlens.hashing.make_hasher (hashing.py:55-64):
    reject empty payloads, never return the reserved value 0."""

    def hash_fn(payload: bytes) -> int:
        if len(payload) == 0:
            raise EmptyPayload()
        return raw(payload) or 1

    return hash_fn


hash_bytes: HashFn = make_hasher(_fold64_device)


def hash_batch(payloads: Sequence) -> list[int]:
    """Digests of many host buffers in one call (b2l_hash_host): contiguous
    buffers are copied in merged DMAs through a double-buffered device ring,
    overlapped with hashing.  Raises EmptyPayload if any payload is empty."""
    n = len(payloads)
    if n == 0:
        return []
    views = [_host_view(p) for p in payloads]
    if any(v[1] == 0 for v in views):
        raise EmptyPayload()
    ptrs = np.array([v[0] for v in views], dtype=np.uint64)
    lens = np.array([v[1] for v in views], dtype=np.uint64)
    out = np.zeros(n, dtype=np.uint64)
    rc = _lib.lib().b2l_hash_host(ptrs.ctypes.data, lens.ctypes.data, n, out.ctypes.data)
    _lib.check(rc, "b2l_hash_host")
    del views
    return [int(x) for x in out]


def hash_host_arrays(ptrs: np.ndarray, lens: np.ndarray, out: np.ndarray) -> None:
    """Columnar host entry: uint64 arrays of host addresses and lengths -> digests (in place)."""
    assert ptrs.dtype == np.uint64 and lens.dtype == np.uint64 and out.dtype == np.uint64
    rc = _lib.lib().b2l_hash_host(ptrs.ctypes.data, lens.ctypes.data, len(ptrs), out.ctypes.data)
    _lib.check(rc, "b2l_hash_host")


def hash_device(ptrs, lens, out, order=None, stream=None) -> None:
    """Raw device batch: int64 CUDA tensors of device addresses / lengths and an
    int64 CUDA tensor for the digests (bit pattern of the u64).  Asynchronous
    on ``stream`` (default: torch's current stream).  A zero length gives
    digest 0 (the reserved "no hash" value)."""
    import torch

    n = ptrs.numel()
    if stream is None:
        stream = torch.cuda.current_stream(ptrs.device)
    sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    order_ptr = order.data_ptr() if order is not None else None
    rc = _lib.lib().b2l_hash_batch(ptrs.data_ptr(), lens.data_ptr(), n, out.data_ptr(), order_ptr, sp)
    _lib.check(rc, "b2l_hash_batch")


K2_MIN_BYTES = 32 << 20  # buffers whose serial chain would dominate: hashed by the whole GPU (K2)
K2_SOLO_BYTES = 96 << 10  # a lone buffer: K2's ~80 us floor beats the 1.6 ns/B serial chain above this


def hash_large(ptr: int, nbytes: int, out_ptr: int, stream=None) -> None:
    """One device buffer (address, length) with the whole GPU -- b2l_hash_large (K2).
    Writes the u64 digest to device address ``out_ptr``.  Asynchronous."""
    import torch
    if nbytes == 0:
        raise EmptyPayload()
    if stream is None:
        stream = torch.cuda.current_stream()
    sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    _lib.check(_lib.lib().b2l_hash_large(ptr, nbytes, out_ptr, sp), "b2l_hash_large")


def hash_large_many(ptrs, lens, out_ptr: int, stream=None) -> None:
    """n huge device buffers (addresses, lengths) -> n u64 digests at device address
    ``out_ptr`` -- b2l_hash_large_many (K2, several buffers per launch).  Asynchronous."""
    import torch
    n = len(ptrs)
    if n == 0:
        return
    if any(int(x) == 0 for x in lens):
        raise EmptyPayload()
    if stream is None:
        stream = torch.cuda.current_stream()
    sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    p = np.ascontiguousarray(np.asarray(ptrs, dtype=np.uint64))
    ln = np.ascontiguousarray(np.asarray(lens, dtype=np.uint64))
    _lib.check(_lib.lib().b2l_hash_large_many(p.ctypes.data, ln.ctypes.data, n, out_ptr, sp), "b2l_hash_large_many")


def hash_tensors(tensors: Sequence, stream=None):
    """Digests of device-resident tensors' bytes, as an int64 CUDA tensor
    holding the u64 bit patterns (``to_u64_list`` converts).  Ragged batches
    are processed longest-first."""
    import torch

    if len(tensors) == 0:
        return torch.zeros(0, dtype=torch.int64)
    dev = tensors[0].device
    lens_h = [t.numel() * t.element_size() for t in tensors]
    if any(n == 0 for n in lens_h):
        raise EmptyPayload()
    for t in tensors:
        if not t.is_contiguous() or t.device != dev:
            raise ValueError("hash_tensors needs contiguous tensors on one CUDA device")
    if stream is not None:  # torch's own copies and scatters below go on the caller's stream too
        if not isinstance(stream, torch.cuda.Stream):
            stream = torch.cuda.ExternalStream(int(stream), device=dev)
        if stream != torch.cuda.current_stream(dev):
            with torch.cuda.stream(stream):
                return hash_tensors(tensors, stream=stream)
    out = torch.empty(len(tensors), dtype=torch.int64, device=dev)
    big = [i for i, n in enumerate(lens_h) if n >= (K2_SOLO_BYTES if len(tensors) == 1 else K2_MIN_BYTES)]
    if big:  # the huge buffers with the whole GPU (K2, several per launch), then the rest as one batch
        bout = torch.empty(len(big), dtype=torch.int64, device=dev)
        hash_large_many([tensors[i].data_ptr() for i in big], [lens_h[i] for i in big], bout.data_ptr(), stream)
        out[torch.tensor(big, device=dev)] = bout
        bigs = set(big)
        small = [i for i in range(len(tensors)) if i not in bigs]
        if small:
            sub = hash_tensors([tensors[i] for i in small], stream=stream)
            out[torch.tensor(small, device=dev)] = sub
        return out
    meta = torch.tensor([[t.data_ptr() for t in tensors], lens_h], dtype=torch.int64)
    order = None
    if len(set(lens_h)) > 1:
        order = torch.from_numpy(np.argsort(-np.asarray(lens_h, dtype=np.int64), kind="stable")
                                 .astype(np.int32)).to(dev, non_blocking=True)
    meta_d = meta.to(dev, non_blocking=True)
    hash_device(meta_d[0], meta_d[1], out, order=order, stream=stream)
    return out


def to_u64_list(t) -> list[int]:
    """int64 digest tensor/array -> Python ints in [0, 2**64)."""
    arr = t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
    return [int(x) & U64_MASK for x in arr.view(np.uint64)]


# ---------------------------------------------------------------------------- collision audit
class CollisionAuditStore:
    """Drop-in for dmlens.hashing.CollisionAuditStore (hashing.py:70-87): keeps the first
    payload per hash, counts byte-unequal repeats.  Observations are buffered and audited on
    the device in one batch (b2l_audit_batch) when ``collision_count`` or ``len()`` is read;
    the result equals observing them one by one."""

    def __init__(self) -> None:
        self._obs: list = []          # (hash, payload bytes) in observation order
        self._count = 0
        self._distinct = 0
        self._clean = True

    def observe(self, hash_value: int, payload: bytes) -> None:
        self._obs.append((int(hash_value), bytes(payload)))
        self._clean = False

    def _flush(self):
        if self._clean:
            return
        self._count, self._distinct = audit_payloads([h for h, _ in self._obs], [p for _, p in self._obs])
        self._clean = True

    @property
    def collision_count(self) -> int:
        self._flush()
        return self._count

    def __len__(self) -> int:
        self._flush()
        return self._distinct


def audit_observe(store: CollisionAuditStore, hash_value: int, payload: bytes) -> CollisionAuditStore:
    store.observe(hash_value, payload)
    return store


def audit_payloads(hashes, payloads) -> tuple:
    """(collision_count, distinct hashes) of observations in order -- host payloads are
    packed into one device slab and audited by b2l_audit_batch."""
    import torch

    n = len(hashes)
    if n == 0:
        return 0, 0
    lens = np.array([len(p) for p in payloads], dtype=np.int64)
    offs = np.zeros(n, dtype=np.int64)
    if n > 1:
        offs[1:] = np.cumsum((lens + 15) // 16 * 16)[:-1]
    total = int(offs[-1] + lens[-1]) + 16
    host = np.zeros(total, dtype=np.uint8)
    for o, p in zip(offs.tolist(), payloads):
        if p:
            host[o:o + len(p)] = np.frombuffer(p, dtype=np.uint8)
    dev = torch.device("cuda", torch.cuda.current_device())
    slab = torch.from_numpy(host).to(dev)
    return audit_device(torch.tensor(np.array(hashes, dtype=np.uint64).view(np.int64), device=dev),
                        torch.from_numpy(offs).to(dev) + slab.data_ptr(), torch.from_numpy(lens).to(dev))


def audit_device(hashes, ptrs, lens) -> tuple:
    """Device observations: int64 CUDA tensors of hash bit patterns, device addresses, lengths."""
    c, d = ctypes.c_uint64(0), ctypes.c_uint64(0)
    L = _lib.lib()
    L.b2l_audit_batch.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    _lib.check(L.b2l_audit_batch(hashes.data_ptr(), ptrs.data_ptr(), lens.data_ptr(), hashes.numel(),
                                 ctypes.byref(c), ctypes.byref(d)), "b2l_audit_batch")
    return int(c.value), int(d.value)
