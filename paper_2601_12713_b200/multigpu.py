"""Multi-GPU hashing (SURVEY.md 8(e) "Hashing": independent buffers shard with no data-path
collective; the only exchange is the 8-byte digests).

One process, several GPUs (the C-level context, include/b2l.h "multi-GPU"):
  init(devices) / shutdown()                   b2l_init / b2l_shutdown
  hash_batch_multi(payloads) -> list[int]      host buffers over every initialised GPU
  hash_host_arrays_multi(ptrs, lens, out)      the same on uint64 address/length arrays

One rank per GPU (torch.distributed, ``sharded.TorchComm``; ``sharded.LocalComm`` for ranks as
threads):
  lpt_partition(lens, parts) -> (owner, load)  LPT placement of a global batch by size
  hash_sharded(ptrs, lens, index, n, comm)     each rank hashes the buffers resident in its HBM,
                                               digests gathered to rank `dst` in global order
  gather_digests(digests, index, n, comm)      just the gather (one exact-size NCCL call)

Per buffer the contract is the reference's (hashing.py:34-67); every digest comes from the
sm_100a kernels in libb2l.so.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .errors import EmptyPayload
from .hashing import _host_view, hash_device


def init(devices: Sequence[int]) -> None:
    devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
    _lib.check(_lib.lib().b2l_init(len(devices), devs), "b2l_init")


def shutdown() -> None:
    _lib.check(_lib.lib().b2l_shutdown(), "b2l_shutdown")


def devices() -> list:
    n = ctypes.c_int(0)
    buf = (ctypes.c_int * 64)()
    _lib.check(_lib.lib().b2l_ngpus(ctypes.byref(n), buf, 64), "b2l_ngpus")
    return [int(buf[i]) for i in range(n.value)]


def lpt_partition(lens, parts: int):
    """LPT placement (longest first, each buffer to the least-loaded part): owner[i] in
    [0, parts) and the bytes placed on each part."""
    ln = np.ascontiguousarray(lens, dtype=np.uint64)
    owner = np.zeros(ln.size, dtype=np.uint32)
    load = np.zeros(parts, dtype=np.uint64)
    _lib.check(_lib.lib().b2l_lpt_partition(ln.ctypes.data if ln.size else None, ln.size, int(parts),
                                            owner.ctypes.data if ln.size else None, load.ctypes.data),
               "b2l_lpt_partition")
    return owner, load


def hash_host_arrays_multi(ptrs: np.ndarray, lens: np.ndarray, out: np.ndarray) -> None:
    assert ptrs.dtype == np.uint64 and lens.dtype == np.uint64 and out.dtype == np.uint64
    _lib.check(_lib.lib().b2l_hash_host_multi(ptrs.ctypes.data, lens.ctypes.data, len(ptrs), out.ctypes.data),
               "b2l_hash_host_multi")


def hash_batch_multi(payloads: Sequence) -> list:
    n = len(payloads)
    if n == 0:
        return []
    views = [_host_view(p) for p in payloads]
    if any(v[1] == 0 for v in views):
        raise EmptyPayload()
    ptrs = np.array([v[0] for v in views], dtype=np.uint64)
    lens = np.array([v[1] for v in views], dtype=np.uint64)
    out = np.zeros(n, dtype=np.uint64)
    hash_host_arrays_multi(ptrs, lens, out)
    del views
    return [int(x) for x in out]


def gather_digests(digests, index, n_total: int, comm, dst: int = 0):
    """Rank-local digests of global buffers `index` -> all n_total digests in global order on
    rank `dst` (int64 tensor of u64 bit patterns; None on the other ranks).  One exact-size
    gather of (index, digest) rows, then a scatter on `dst`."""
    import torch
    rows = torch.stack([index.to(torch.int64), digests.to(torch.int64)], dim=1)
    got = comm.gatherv(rows, dst)
    if got is None:
        return None
    out = torch.zeros(n_total, dtype=torch.int64, device=got.device)
    out[got[:, 0]] = got[:, 1]
    return out


def hash_sharded(ptrs, lens, index, n_total: int, comm, dst: int = 0, order=None, stream=None):
    """Each rank hashes its resident buffers (int64 CUDA tensors of device addresses / lengths;
    `index` = their global buffer ids), then the digests are gathered to rank `dst` in global
    order.  Returns the full digest tensor on `dst`, None elsewhere."""
    import torch
    out = torch.empty(ptrs.numel(), dtype=torch.int64, device=ptrs.device)
    if ptrs.numel():
        hash_device(ptrs, lens, out, order=order, stream=stream)
    return gather_digests(out, index, n_total, comm, dst)
