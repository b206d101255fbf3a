"""Key-range sharded trace analysis across G ranks.

Input: rank r holds a seq-range shard of the trace (contiguous events
[base_r, base_r + n_r)).  The detectors split along two keys:

  * hash-keyed work -- DD and RT (detectors.py:85-167) only ever relate
    transfers with the same content hash, so hashed transfers go to the rank
    owning their hash range ((hash * G) >> 64);
  * device-keyed work -- LIFO pairing (prep.py:45-96, key (dst_dev, dst_addr)),
    RA (key (src_addr, dst_dev, bytes)), UA and UT (per target device sweeps,
    detectors.py:194-271) never cross a device, so allocs/deletes, target
    kernels and target transfers go to the rank owning their device (dev % G).

One all-to-all redistributes the events (both key spaces in one exchange);
each rank runs the single-GPU engine on its two sub-traces (a sub-trace keeps
global trace order, so every detector is exact on it; the synthetic-delete
time, a trace-wide max, comes from one all-reduce); a final gather brings the
findings to rank 0, which merges them into the reference's global orders
(groups by (first start, key...), pairs by allocation, lists by position).

The exchange goes through a small communicator interface: ``TorchComm``
(torch.distributed: NCCL on GPUs, gloo on CPU) or ``LocalComm`` (G ranks as
threads of one process -- used to check G-way parity on a single GPU).
"""
from __future__ import annotations

import threading
from typing import Callable, List, Optional

import numpy as np

from .analysis import FLAG_SKIP_ALLOC, FLAG_SKIP_DDRT, FLAG_VALIDATE_ONLY, ColumnarFindings, EngineInvalid
from .columns import Columns

FIELDS = ("seq", "start_ns", "end_ns", "src_addr", "dst_addr", "bytes", "hash", "src_device", "dst_device",
          "kind", "loc")
ROW = 1 + len(FIELDS)  # global index + fields, one u64 each
SYN = np.uint32(0xFFFFFFFF)
TRANSFER, ALLOC, DELETE, KERNEL = 0, 1, 2, 3


# ------------------------------------------------------------------------ communicators
class LocalComm:
    """G ranks as threads of one process (shared slots + a barrier)."""

    class _Shared:
        def __init__(self, g):
            self.g = g
            self.barrier = threading.Barrier(g)
            self.slots = [None] * g

    def __init__(self, shared, rank):
        self.s, self.rank, self.size = shared, rank, shared.g

    @classmethod
    def group(cls, g):
        sh = cls._Shared(g)
        return [cls(sh, r) for r in range(g)]

    def _exchange(self, obj):
        self.s.barrier.wait()
        self.s.slots[self.rank] = obj
        self.s.barrier.wait()
        out = list(self.s.slots)
        self.s.barrier.wait()
        return out

    def alltoall(self, parts: List[np.ndarray]) -> List[np.ndarray]:
        allp = self._exchange(parts)
        return [allp[src][self.rank] for src in range(self.size)]

    def allreduce_max(self, v: int) -> int:
        return max(self._exchange(int(v)))

    def alltoall_rows(self, rows, counts):
        """Device rows grouped by destination rank (counts[r] rows for rank r) -> the rows every
        rank sent to this one, in rank order (torch tensors stay on the device)."""
        import torch
        allp = self._exchange((rows, [int(x) for x in counts]))
        got = []
        for src_rows, src_counts in allp:
            o = sum(src_counts[:self.rank])
            got.append(src_rows[o:o + src_counts[self.rank]])
        return torch.cat(got) if got else rows[:0]

    def allgather(self, obj):
        return self._exchange(obj)

    def gather0(self, obj):
        out = self._exchange(obj)
        return out if self.rank == 0 else None

    def gather0_findings(self, out: dict):
        return self.gather0(out)

    def gatherv(self, t, dst: int = 0):
        """Tensors of any length (same trailing shape) -> their concatenation in rank order on
        `dst` (None elsewhere); stays on the tensors' device."""
        import torch
        if t.is_cuda:  # another thread's stream reads it next
            torch.cuda.current_stream(t.device).synchronize()
        allp = self._exchange(t)
        return torch.cat(allp) if self.rank == dst else None


class TorchComm:
    """torch.distributed communicator (NCCL for CUDA tensors, gloo on CPU)."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.dist, self.torch = dist, torch
        self.rank, self.size = dist.get_rank(), dist.get_world_size()
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu"))

    def alltoall(self, parts: List[np.ndarray]) -> List[np.ndarray]:
        torch = self.torch
        sizes = torch.tensor([p.shape[0] for p in parts], dtype=torch.int64, device=self.device)
        rsizes = torch.empty_like(sizes)
        self.dist.all_to_all_single(rsizes, sizes)
        rs = rsizes.cpu().tolist()
        send = np.concatenate([p.reshape(-1, ROW) for p in parts]).view(np.int64) if parts else np.zeros((0, ROW))
        st = torch.from_numpy(np.ascontiguousarray(send).reshape(-1)).to(self.device)
        rt = torch.empty(sum(rs) * ROW, dtype=torch.int64, device=self.device)
        self.dist.all_to_all_single(rt, st, [r * ROW for r in rs], [p.shape[0] * ROW for p in parts])
        flat = rt.cpu().numpy().view(np.uint64).reshape(-1, ROW)
        out, o = [], 0
        for r in rs:
            out.append(flat[o:o + r])
            o += r
        return out

    def alltoall_rows(self, rows, counts):
        """Device rows grouped by destination rank -> rows received from every rank, in rank order:
        one all_to_all_single of the sizes, one of the rows (NCCL moves device memory over
        NVLink; gloo stages through host memory)."""
        torch, dist = self.torch, self.dist
        width = rows.shape[1]
        sizes = torch.tensor([int(x) for x in counts], dtype=torch.int64, device=self.device)
        rsizes = torch.empty_like(sizes)
        dist.all_to_all_single(rsizes, sizes)
        rs = rsizes.cpu().tolist()
        send = rows if self.device.type == rows.device.type else rows.to(self.device)
        recv = torch.empty((sum(rs), width), dtype=rows.dtype, device=self.device)
        dist.all_to_all_single(recv.view(-1), send.reshape(-1), [r * width for r in rs],
                               [int(c) * width for c in counts])
        return recv if recv.device == rows.device else recv.to(rows.device)

    def allreduce_max(self, v: int) -> int:
        """Max of a u64 over ranks, as (hi, lo) 32-bit halves (exact for any u64)."""
        torch, dist = self.torch, self.dist
        hi = torch.tensor([int(v) >> 32], dtype=torch.int64, device=self.device)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        mine = (int(v) & 0xFFFFFFFF) if (int(v) >> 32) == int(hi.item()) else 0
        lo = torch.tensor([mine], dtype=torch.int64, device=self.device)
        dist.all_reduce(lo, op=dist.ReduceOp.MAX)
        return (int(hi.item()) << 32) | int(lo.item())

    def allgather(self, obj):
        out = [None] * self.size
        self.dist.all_gather_object(out, obj)
        return out

    def gather0(self, obj):
        out = [None] * self.size if self.rank == 0 else None
        self.dist.gather_object(obj, out, dst=0)
        return out

    def gatherv(self, t, dst: int = 0):
        """Exact-size gather: tensors of any length (same trailing shape) -> their concatenation in
        rank order on `dst` (None elsewhere).  One size all-gather, then one all_to_all_single in
        which only `dst` receives (NCCL moves device memory; no padding)."""
        torch, dist = self.torch, self.dist
        width = int(np.prod(t.shape[1:])) if t.dim() > 1 else 1
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=self.device)
        ns = [torch.empty_like(n) for _ in range(self.size)]
        dist.all_gather(ns, n)
        sizes = [int(x.item()) for x in ns]
        send = t if t.device.type == self.device.type else t.to(self.device)
        send = send.contiguous().view(-1)
        rows = sum(sizes) if self.rank == dst else 0
        recv = torch.empty(rows * width, dtype=t.dtype, device=self.device)
        in_split = [t.shape[0] * width if r == dst else 0 for r in range(self.size)]
        out_split = [sz * width if self.rank == dst else 0 for sz in sizes]
        dist.all_to_all_single(recv, send, out_split, in_split)
        if self.rank != dst:
            return None
        recv = recv.view(rows, *t.shape[1:]) if t.dim() > 1 else recv
        return recv if recv.device == t.device else recv.to(t.device)

    def gather0_findings(self, out: dict):
        """Per-rank findings (dict of numpy arrays / tuples of arrays) to rank 0 as ONE flat int64
        tensor per rank (a size all-gather, then one all-gather of padded buffers; NCCL moves
        device memory) instead of pickled objects."""
        torch, dist = self.torch, self.dist
        flat = _pack_findings(out)
        n = torch.tensor([flat.size], dtype=torch.int64, device=self.device)
        ns = [torch.empty_like(n) for _ in range(self.size)]
        dist.all_gather(ns, n)
        sizes = [int(x.item()) for x in ns]
        buf = torch.zeros(max(sizes), dtype=torch.int64, device=self.device)
        buf[:flat.size] = torch.from_numpy(flat).to(self.device)
        bufs = [torch.empty_like(buf) for _ in range(self.size)]
        dist.all_gather(bufs, buf)
        if self.rank != 0:
            return None
        return [_unpack_findings(b[:sz].cpu().numpy()) for b, sz in zip(bufs, sizes)]


# ------------------------------------------------------------------------ findings wire format
# Per-rank findings as one int64 array: [n_fields, (key id, slot, dtype id, length) * n_fields,
# payloads (each widened to 64-bit lanes)].  Keys are the detector names of analyze_sharded_device.
_FKEYS = ("dd", "rt", "pairs", "warn", "ra", "ua", "ut")
_FDTYPES = (np.int64, np.uint64, np.int32, np.uint32)


def _pack_findings(out: dict) -> np.ndarray:
    fields = []
    for ki, key in enumerate(_FKEYS):
        if key not in out:
            continue
        val = out[key]
        arrs = val if isinstance(val, tuple) else (val,)
        for slot, a in enumerate(arrs):
            a = np.ascontiguousarray(a)
            di = next(i for i, d in enumerate(_FDTYPES) if a.dtype == d)
            slot_id = slot if isinstance(val, tuple) else -1
            fields.append((ki, slot_id, di, a))
    head = [len(fields)]
    for ki, slot, di, a in fields:
        head += [ki, slot, di, a.size]
    body = [a.astype(np.int64) if a.dtype != np.uint64 else a.view(np.int64) for _, _, _, a in fields]
    return np.concatenate([np.asarray(head, dtype=np.int64)] + body) if body else np.asarray(head, np.int64)


def _unpack_findings(flat: np.ndarray) -> dict:
    nf = int(flat[0])
    head = flat[1:1 + 4 * nf].reshape(nf, 4)
    o = 1 + 4 * nf
    out: dict = {}
    for ki, slot, di, ln in head.tolist():
        seg = flat[o:o + ln]
        o += ln
        d = _FDTYPES[di]
        a = seg.view(np.uint64).copy() if d == np.uint64 else seg.astype(d)
        key = _FKEYS[ki]
        if slot < 0:
            out[key] = a
        else:
            out.setdefault(key, []).append(a)
    return {k: (tuple(v) if isinstance(v, list) else v) for k, v in out.items()}


# ------------------------------------------------------------------------ packing
def _rows(cols: Columns, idx: np.ndarray, base: int) -> np.ndarray:
    r = np.empty((idx.size, ROW), dtype=np.uint64)
    r[:, 0] = idx.astype(np.uint64) + np.uint64(base)
    for k, f in enumerate(FIELDS):
        a = getattr(cols, f)[idx]
        r[:, k + 1] = a.astype(np.int64).view(np.uint64) if a.dtype == np.int32 else a.astype(np.uint64)
    return r


def _subtrace(rows: np.ndarray, like: Columns):
    g = rows[:, 0].astype(np.int64)
    order = np.argsort(g, kind="stable")  # concatenation of rank-ordered runs is already sorted; be safe
    rows = rows[order]
    col = {}
    for k, f in enumerate(FIELDS):
        v = rows[:, k + 1]
        col[f] = v.view(np.int64).astype(np.int32) if f in ("src_device", "dst_device") else (
            v.astype(np.uint8) if f == "kind" else (v.astype(np.uint32) if f == "loc" else v.copy()))
    sub = Columns(n=rows.shape[0], num_devices_total=like.num_devices_total, host_device=like.host_device,
                  seq=col["seq"], start_ns=col["start_ns"], end_ns=col["end_ns"], src_addr=col["src_addr"],
                  dst_addr=col["dst_addr"], bytes=col["bytes"], hash=col["hash"], src_device=col["src_device"],
                  dst_device=col["dst_device"], kind=col["kind"], loc=col["loc"], loc_flags=like.loc_flags,
                  loc_bucket=like.loc_bucket, n_buckets=like.n_buckets, bucket_keys=like.bucket_keys,
                  wall_time_ns=like.wall_time_ns, locs=like.locs)
    return sub, rows[:, 0].astype(np.int64)


def hash_owner(h: np.ndarray, g: int) -> np.ndarray:
    return (((h >> np.uint64(32)) * np.uint64(g)) >> np.uint64(32)).astype(np.int64)


# ------------------------------------------------------------------------ the sharded pipeline
def engine_analyzer(cols, flags=0, synthetic_end_ns=None, strict=False):
    from .analysis import analyze_columns
    return analyze_columns(cols, strict=strict, flags=flags, synthetic_end_ns=synthetic_end_ns)


def analyze_sharded(shard: Columns, base: int, comm, strict: bool = False,
                    analyzer: Callable = engine_analyzer) -> Optional[ColumnarFindings]:
    """Findings of the whole trace (global event indices) on rank 0, None elsewhere.
    Raises EngineInvalid (global indices) on every rank if any shard fails validation."""
    G = comm.size
    # ---- 1. validation of every shard + the order rule across shard boundaries (model.py:193-196)
    bad_i, bad_r = np.zeros(0, np.int64), np.zeros(0, np.uint32)
    try:
        analyzer(shard, flags=FLAG_VALIDATE_ONLY)
    except EngineInvalid as exc:
        bad_i, bad_r = exc.bad_index.astype(np.int64), exc.bad_rules.astype(np.uint32)
    edge = (int(shard.start_ns[0]), int(shard.seq[0]), int(shard.start_ns[-1]), int(shard.seq[-1])) \
        if shard.n else None
    edges = comm.allgather(edge)
    prev = None
    for r in range(comm.rank):
        if edges[r] is not None:
            prev = edges[r]
    if prev is not None and shard.n:
        s0, q0 = int(shard.start_ns[0]), int(shard.seq[0])
        m = 0
        if s0 < prev[2] or (s0 == prev[2] and q0 < prev[3]):
            m |= 1 << 10
        if q0 <= prev[3]:
            m |= 1 << 11
        if m:
            k = np.nonzero(bad_i == 0)[0]
            if k.size:
                bad_r[k[0]] |= m
            else:
                bad_i, bad_r = np.concatenate([[0], bad_i]), np.concatenate([[m], bad_r]).astype(np.uint32)
    all_bad = comm.allgather((bad_i + base, bad_r))
    gi = np.concatenate([b[0] for b in all_bad])
    if gi.size:
        raise EngineInvalid(gi.astype(np.uint32), np.concatenate([b[1] for b in all_bad]).astype(np.uint32))

    # ---- 2. one all-to-all: hashed transfers by hash range, device work by device
    kind, nb, h, dst = shard.kind, shard.bytes, shard.hash, shard.dst_device.astype(np.int64)
    is_h = (kind == TRANSFER) & (nb > 0) & (h != 0)
    is_d = (kind == ALLOC) | (kind == DELETE) | (((kind == KERNEL) | (kind == TRANSFER)) & (dst != shard.host_device))
    dmax = int(shard.end_ns[kind != KERNEL].max()) if np.any(kind != KERNEL) else 0
    ih, idv = np.nonzero(is_h)[0], np.nonzero(is_d)[0]
    oh, od = hash_owner(h[ih], G), dst[idv] % G
    rows_h, rows_d = _rows(shard, ih, base), _rows(shard, idv, base)
    parts = []
    for r in range(G):
        a, b = rows_h[oh == r], rows_d[od == r]
        tag = np.zeros((a.shape[0] + b.shape[0], 1), dtype=np.uint64)
        tag[a.shape[0]:] = 1
        # the tag (key space) travels in the top bit of the global index column
        both = np.concatenate([a, b])
        both[:, 0] |= tag[:, 0] << np.uint64(63)
        parts.append(both)
    got = comm.alltoall(parts)
    synth_end = comm.allreduce_max(dmax)
    rec = np.concatenate(got) if got else np.zeros((0, ROW), np.uint64)
    space = rec[:, 0] >> np.uint64(63)
    rec = rec.copy()
    rec[:, 0] &= np.uint64((1 << 63) - 1)
    sub_h, gid_h = _subtrace(rec[space == 0], shard)
    sub_d, gid_d = _subtrace(rec[space == 1], shard)

    # ---- 3. per-rank engine runs on the two sub-traces
    out = {}
    if sub_h.n:
        f = analyzer(sub_h, flags=FLAG_SKIP_ALLOC, strict=strict)
        G_ = gid_h
        off = f.dd_offsets.astype(np.int64)
        mem = G_[f.dd_members.astype(np.int64)]
        first = mem[off[:-1]] if off.size > 1 else np.zeros(0, np.int64)
        out["dd"] = (off, mem, sub_h.start_ns[f.dd_members[off[:-1]]] if off.size > 1 else np.zeros(0, np.uint64),
                     sub_h.hash[f.dd_members[off[:-1]]] if off.size > 1 else np.zeros(0, np.uint64),
                     sub_h.dst_device[f.dd_members[off[:-1]]] if off.size > 1 else np.zeros(0, np.int32), first)
        off = f.rt_offsets.astype(np.int64)
        tx, rx = f.rt_tx.astype(np.int64), f.rt_rx.astype(np.int64)
        ft = tx[off[:-1]] if off.size > 1 else np.zeros(0, np.int64)
        out["rt"] = (off, G_[tx], G_[rx], sub_h.start_ns[ft], sub_h.hash[ft], sub_h.src_device[ft],
                     sub_h.dst_device[ft])
    if sub_d.n:
        f = analyzer(sub_d, flags=FLAG_SKIP_DDRT, synthetic_end_ns=synth_end)
        G_ = gid_d
        pa = f.pair_alloc.astype(np.int64)
        pd = f.pair_delete
        out["pairs"] = (G_[pa], np.where(pd == SYN, -1, G_[np.where(pd == SYN, 0, pd).astype(np.int64)]))
        out["warn"] = G_[f.warn_index.astype(np.int64)]
        off = f.ra_offsets.astype(np.int64)
        ra_alloc = G_[pa[f.ra_pairs.astype(np.int64)]]
        fa = pa[f.ra_pairs[off[:-1]].astype(np.int64)] if off.size > 1 else np.zeros(0, np.int64)
        out["ra"] = (off, ra_alloc, sub_d.start_ns[fa], sub_d.src_addr[fa], sub_d.dst_device[fa], sub_d.bytes[fa])
        out["ua"] = G_[pa[f.ua_pairs.astype(np.int64)]]
        out["ut"] = G_[f.ut_events.astype(np.int64)]
    parts = comm.gather0(out)
    if comm.rank != 0:
        return None
    return _merge(parts, synth_end, total_events=None)


# ------------------------------------------------------------------------ device-resident pipeline
_SHARD_FIELDS = ("gid", "seq", "start_ns", "end_ns", "src_addr", "dst_addr", "bytes", "hash", "src_device",
                 "dst_device", "kind", "loc")


def _shard_lib():
    import ctypes

    from . import _lib
    L = _lib.lib()
    L.b2l_shard_route.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    L.b2l_shard_unpack.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                   ctypes.c_void_p]
    return L, _lib


def _route(shard, base: int, G: int):
    """b2l_shard_route: device rows grouped by destination rank, counts, max data-op end."""
    import ctypes

    import torch
    L, _lib = _shard_lib()
    dev = shard.t["seq"].device
    rows = torch.empty((max(2 * shard.n, 1), ROW), dtype=torch.int64, device=dev)
    counts = np.zeros(G, np.uint64)
    nrec, dend = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _lib.check(L.b2l_shard_route(ctypes.addressof(shard.struct), G, base, 0, rows.data_ptr(), counts.ctypes.data,
                                 ctypes.addressof(nrec), ctypes.addressof(dend)), "b2l_shard_route")
    return rows[:nrec.value], counts, int(dend.value)


def _unpack(recv, space: int, like):
    """Rows of one key space -> (DeviceColumns sub-trace, global indices as a device tensor)."""
    import ctypes

    import torch

    from .analysis import DeviceColumns
    L, _lib = _shard_lib()
    m, dev = recv.shape[0], recv.device
    dt = {"src_device": torch.int32, "dst_device": torch.int32, "kind": torch.uint8, "loc": torch.int32}
    t = {f: torch.empty(max(m, 1), dtype=dt.get(f, torch.int64), device=dev) for f in _SHARD_FIELDS}
    ptrs = (ctypes.c_void_p * len(_SHARD_FIELDS))(*[t[f].data_ptr() for f in _SHARD_FIELDS])
    n = ctypes.c_uint64(0)
    _lib.check(L.b2l_shard_unpack(recv.data_ptr() if m else None, m, space, ptrs, ctypes.addressof(n)),
               "b2l_shard_unpack")
    k = n.value
    gid = t.pop("gid")[:k]
    return DeviceColumns.from_device({f: v[:k] for f, v in t.items()}, k, like), gid


def _host(tensor, idx: np.ndarray, dtype):
    """Device column values at host indices (small gathers for group sort keys)."""
    import torch
    if idx.size == 0:
        return np.zeros(0, dtype)
    ii = torch.from_numpy(np.ascontiguousarray(idx.astype(np.int64))).to(tensor.device)
    v = tensor[ii].cpu().numpy()
    return v.view(dtype) if v.dtype.itemsize == np.dtype(dtype).itemsize else v.astype(dtype)


class _Phases:
    """B2L_SHARD_TRACE=1: wall time of each phase on rank 0 (diagnostics only)."""

    def __init__(self, rank):
        import os
        import time
        self.on = rank == 0 and os.environ.get("B2L_SHARD_TRACE") is not None
        self.time = time
        self.t = time.perf_counter()

    def mark(self, name):
        if self.on:
            now = self.time.perf_counter()
            print(f"[shard] {name:10s} {1e3 * (now - self.t):8.3f} ms", flush=True)
            self.t = now


def analyze_sharded_device(shard, base: int, comm, strict: bool = False, gather: bool = True):
    """The sharded pipeline with every event-sized step on the device: ``shard`` is a
    DeviceColumns seq-range shard; validation, routing (b2l_shard_route), the all-to-all of
    the rows (NCCL on device memory), unpacking (b2l_shard_unpack) and both engine runs stay in
    HBM.  Only the findings (global indices and group sort keys) travel to rank 0 for the merge.
    Same results and exceptions as ``analyze_sharded``.  ``gather=False`` stops before the gather:
    every rank returns its own key range's findings (the per-rank parts, global indices)."""
    from .analysis import analyze_columns
    G = comm.size
    host = shard.host
    ph = _Phases(comm.rank)
    # ---- 1. validation (engine on the device shard) + the order rule across shard boundaries
    bad_i, bad_r = np.zeros(0, np.int64), np.zeros(0, np.uint32)
    try:
        analyze_columns(shard, flags=FLAG_VALIDATE_ONLY)
    except EngineInvalid as exc:
        bad_i, bad_r = exc.bad_index.astype(np.int64), exc.bad_rules.astype(np.uint32)
    edge = (int(host.start_ns[0]), int(host.seq[0]), int(host.start_ns[-1]), int(host.seq[-1])) if host.n else None
    edges = comm.allgather(edge)
    prev = None
    for r in range(comm.rank):
        if edges[r] is not None:
            prev = edges[r]
    if prev is not None and host.n:
        s0, q0 = int(host.start_ns[0]), int(host.seq[0])
        m = 0
        if s0 < prev[2] or (s0 == prev[2] and q0 < prev[3]):
            m |= 1 << 10
        if q0 <= prev[3]:
            m |= 1 << 11
        if m:
            k = np.nonzero(bad_i == 0)[0]
            if k.size:
                bad_r[k[0]] |= m
            else:
                bad_i, bad_r = np.concatenate([[0], bad_i]), np.concatenate([[m], bad_r]).astype(np.uint32)
    all_bad = comm.allgather((bad_i + base, bad_r))
    gi = np.concatenate([b[0] for b in all_bad])
    if gi.size:
        raise EngineInvalid(gi.astype(np.uint32), np.concatenate([b[1] for b in all_bad]).astype(np.uint32))
    ph.mark("validate")
    # ---- 2. route + one all-to-all of device rows
    rows, counts, dmax = _route(shard, base, G) if host.n else (None, np.zeros(G, np.uint64), 0)
    if rows is None:
        import torch
        rows = torch.empty((0, ROW), dtype=torch.int64, device=shard.t["seq"].device)
    ph.mark("route")
    recv = comm.alltoall_rows(rows, counts)
    synth_end = comm.allreduce_max(dmax)
    ph.mark("exchange")
    sub_h, gid_h = _unpack(recv, 0, shard)
    sub_d, gid_d = _unpack(recv, 1, shard)
    ph.mark("unpack")
    # ---- 3. per-rank engine runs on the two device sub-traces
    out = {}
    if sub_h.n:
        f = analyzer_dev(sub_h, flags=FLAG_SKIP_ALLOC, strict=strict)
        G_ = gid_h.cpu().numpy()
        off = f.dd_offsets.astype(np.int64)
        mem_l = f.dd_members.astype(np.int64)
        fl = mem_l[off[:-1]] if off.size > 1 else np.zeros(0, np.int64)
        t = sub_h.t
        out["dd"] = (off, G_[mem_l], _host(t["start_ns"], fl, np.uint64), _host(t["hash"], fl, np.uint64),
                     _host(t["dst_device"], fl, np.int32), G_[fl])
        off = f.rt_offsets.astype(np.int64)
        tx, rx = f.rt_tx.astype(np.int64), f.rt_rx.astype(np.int64)
        ft = tx[off[:-1]] if off.size > 1 else np.zeros(0, np.int64)
        out["rt"] = (off, G_[tx], G_[rx], _host(t["start_ns"], ft, np.uint64), _host(t["hash"], ft, np.uint64),
                     _host(t["src_device"], ft, np.int32), _host(t["dst_device"], ft, np.int32))
    if sub_d.n:
        f = analyzer_dev(sub_d, flags=FLAG_SKIP_DDRT, synthetic_end_ns=synth_end)
        G_ = gid_d.cpu().numpy()
        pa = f.pair_alloc.astype(np.int64)
        pd = f.pair_delete
        out["pairs"] = (G_[pa], np.where(pd == SYN, -1, G_[np.where(pd == SYN, 0, pd).astype(np.int64)]))
        out["warn"] = G_[f.warn_index.astype(np.int64)]
        off = f.ra_offsets.astype(np.int64)
        ra_alloc = G_[pa[f.ra_pairs.astype(np.int64)]]
        fa = pa[f.ra_pairs[off[:-1]].astype(np.int64)] if off.size > 1 else np.zeros(0, np.int64)
        t = sub_d.t
        out["ra"] = (off, ra_alloc, _host(t["start_ns"], fa, np.uint64), _host(t["src_addr"], fa, np.uint64),
                     _host(t["dst_device"], fa, np.int32), _host(t["bytes"], fa, np.uint64))
        out["ua"] = G_[pa[f.ua_pairs.astype(np.int64)]]
        out["ut"] = G_[f.ut_events.astype(np.int64)]
    ph.mark("engine")
    if not gather:
        return out
    parts = comm.gather0_findings(out) if hasattr(comm, "gather0_findings") else comm.gather0(out)
    ph.mark("gather")
    if comm.rank != 0:
        return None
    res = _merge_dev(parts, synth_end, shard.t["seq"].device)
    ph.mark("merge")
    return res


def analyzer_dev(cols, flags=0, synthetic_end_ns=None, strict=False):
    from .analysis import analyze_columns
    return analyze_columns(cols, strict=strict, flags=flags, synthetic_end_ns=synthetic_end_ns)


def _cat(parts, key, k, dtype):
    arrs = [p[key][k] for p in parts if key in p]
    return np.concatenate(arrs).astype(dtype) if arrs else np.zeros(0, dtype)


def _np_lexsort(kcols):
    return np.lexsort(tuple(reversed(kcols)))  # first column is the primary key


def runs_lexsort(kcols):
    """Lexicographic order of key columns (first = primary) for a concatenation of per-rank runs
    that are each already sorted: a stable sort of the primary key alone (timsort merges the
    runs in O(n log G)), then a full lexsort only when the primary key has ties."""
    k0 = kcols[0]
    order = np.argsort(k0, kind="stable")
    s0 = k0[order]
    if s0.size > 1 and np.any(s0[1:] == s0[:-1]):
        return np.lexsort(tuple(reversed(kcols)))
    return order


def _merge_groups(parts, key, member_cols, sort_cols, lexsort=_np_lexsort):
    """Concatenate per-rank groups and order them by the given key columns (lexicographic)."""
    offs, mems, keys = [], [[] for _ in member_cols], [[] for _ in sort_cols]
    for p in parts:
        if key not in p:
            continue
        t = p[key]
        offs.append(t[0])
        for j, c in enumerate(member_cols):
            mems[j].append(t[c])
        for j, c in enumerate(sort_cols):
            keys[j].append(np.asarray(t[c]).astype(np.int64).astype(np.uint64) if np.asarray(t[c]).dtype == np.int32
                           else np.asarray(t[c]).astype(np.uint64))
    sizes = [np.diff(o) for o in offs]
    if not sizes or sum(s.size for s in sizes) == 0:
        return np.zeros(1, np.uint64), [np.zeros(0, np.int64) for _ in member_cols]
    size = np.concatenate(sizes)
    starts = np.concatenate([o[:-1] + sum(len(m) for m in mems[0][:i]) for i, o in enumerate(offs)])
    kcols = [np.concatenate(k) for k in keys]
    order = lexsort(kcols)
    flat = [np.concatenate(m) for m in mems]
    new_off = np.zeros(size.size + 1, np.uint64)
    new_off[1:] = np.cumsum(size[order])
    if order.size:  # members of the groups in their new order (vectorised ranges)
        sz, st = size[order].astype(np.int64), starts[order].astype(np.int64)
        first = np.zeros(sz.size, np.int64)
        first[1:] = np.cumsum(sz)[:-1]
        idx = np.repeat(st - first, sz) + np.arange(int(sz.sum()), dtype=np.int64)
    else:
        idx = np.zeros(0, np.int64)
    return new_off, [f[idx] for f in flat]


def _merge(parts, synth_end, total_events=None, lexsort=_np_lexsort) -> ColumnarFindings:
    dd_off, (dd_mem,) = _merge_groups(parts, "dd", [1], [2, 3, 4], lexsort)
    rt_off, (rt_tx, rt_rx) = _merge_groups(parts, "rt", [1, 2], [3, 4, 5, 6], lexsort)
    pa = _cat(parts, "pairs", 0, np.int64)
    pdl = _cat(parts, "pairs", 1, np.int64)
    o = np.argsort(pa, kind="stable")
    pa, pdl = pa[o], pdl[o]
    ra_off, (ra_alloc,) = _merge_groups(parts, "ra", [1], [2, 3, 4, 5], lexsort)
    # pair rank of an alloc event: a direct lookup table over event ids (random queries into a
    # sorted array would be one cache miss per binary-search step)
    pos = np.zeros(int(pa[-1]) + 1 if pa.size else 1, np.int64)
    pos[pa] = np.arange(pa.size, dtype=np.int64)
    ra_pairs = pos[np.asarray(ra_alloc, dtype=np.int64)]
    ua_ev = np.concatenate([p["ua"] for p in parts if "ua" in p]).astype(np.int64) if any(
        "ua" in p for p in parts) else np.zeros(0, np.int64)
    ua = np.sort(pos[ua_ev])
    ut = np.sort(np.concatenate([p["ut"] for p in parts if "ut" in p])) if any("ut" in p for p in parts) else \
        np.zeros(0, np.int64)
    warn = np.sort(np.concatenate([p["warn"] for p in parts if "warn" in p])) if any(
        "warn" in p for p in parts) else np.zeros(0, np.int64)
    u32 = lambda a: np.asarray(a).astype(np.uint32)  # noqa: E731
    return ColumnarFindings(
        n_events=total_events or 0, dd_offsets=dd_off.astype(np.uint64), dd_members=u32(dd_mem),
        rt_offsets=rt_off.astype(np.uint64), rt_tx=u32(rt_tx), rt_rx=u32(rt_rx), pair_alloc=u32(pa),
        pair_delete=np.where(pdl < 0, SYN, pdl).astype(np.uint32), synthetic_end_ns=int(synth_end),
        warn_index=u32(warn), ra_offsets=ra_off.astype(np.uint64), ra_pairs=u32(ra_pairs), ua_pairs=u32(ua),
        ut_events=u32(ut))


# ------------------------------------------------------------------------ merge on the device
def _dev_lexsort(kcols, dev):
    """Order of u64 key columns (first = primary) as LSD passes of the engine's stable pair
    sort on device arrays (b2l_sort_u64_pairs_device): (k[-2], k[-1]) first, then (k[-4], k[-3])."""
    import ctypes

    import torch

    from . import _lib
    L = _lib.lib()
    L.b2l_sort_u64_pairs_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    n = kcols[0].numel()
    order = torch.arange(n, dtype=torch.int64, device=dev)
    if n < 2:
        return order
    cols = list(kcols)
    if len(cols) % 2:
        cols = [torch.zeros(n, dtype=torch.int64, device=dev)] + cols
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    for j in range(len(cols) - 2, -1, -2):
        a = cols[j][order].contiguous()
        b = cols[j + 1][order].contiguous()
        torch.cuda.synchronize(dev)
        _lib.check(L.b2l_sort_u64_pairs_device(a.data_ptr(), b.data_ptr(), n, perm.data_ptr()),
                   "b2l_sort_u64_pairs_device")
        order = order[perm.long()]
    return order


def _dev(a, dev):
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a.astype(np.int64, copy=False)).to(dev, non_blocking=False)


def _merge_groups_dev(parts, key, member_cols, sort_cols, dev):
    """_merge_groups with the concatenated groups on the device: one engine sort for the order,
    the member ranges gathered with a repeat/arange index."""
    import torch
    offs = [np.asarray(p[key][0], np.int64) for p in parts if key in p]
    if not offs or sum(o.size - 1 for o in offs) == 0:
        return np.zeros(1, np.uint64), [np.zeros(0, np.int64) for _ in member_cols]
    sizes = np.concatenate([np.diff(o) for o in offs])
    base = np.cumsum([0] + [int(o[-1]) for o in offs[:-1]])
    starts = np.concatenate([o[:-1] + b for o, b in zip(offs, base)])
    keys = [_dev(np.concatenate([np.asarray(p[key][c]).astype(np.int64) for p in parts if key in p]), dev)
            for c in sort_cols]
    order = _dev_lexsort(keys, dev)
    sz, st = _dev(sizes, dev)[order], _dev(starts, dev)[order]
    first = torch.cumsum(sz, 0) - sz
    total = int(sizes.sum())
    idx = torch.repeat_interleave(st - first, sz, output_size=total) + torch.arange(total, device=dev)
    new_off = np.zeros(sizes.size + 1, np.uint64)
    new_off[1:] = np.cumsum(sz.cpu().numpy())
    flat = [_dev(np.concatenate([np.asarray(p[key][c]) for p in parts if key in p]), dev)[idx].cpu().numpy()
            for c in member_cols]
    return new_off, flat


def _merge_dev(parts, synth_end, dev) -> ColumnarFindings:
    """_merge on rank 0's GPU: group orders by the engine's radix sort, index work as device
    gathers; same results as the host merge."""
    import torch
    dd_off, (dd_mem,) = _merge_groups_dev(parts, "dd", [1], [2, 3, 4], dev)
    rt_off, (rt_tx, rt_rx) = _merge_groups_dev(parts, "rt", [1, 2], [3, 4, 5, 6], dev)
    pa_h = _cat(parts, "pairs", 0, np.int64)
    pa = _dev(pa_h, dev)
    pdl = _dev(_cat(parts, "pairs", 1, np.int64), dev)
    o = _dev_lexsort([pa], dev)
    pa, pdl = pa[o], pdl[o]
    ra_off, (ra_alloc,) = _merge_groups_dev(parts, "ra", [1], [2, 3, 4, 5], dev)
    pos = torch.zeros(int(pa_h.max()) + 1 if pa_h.size else 1, dtype=torch.int64, device=dev)
    pos[pa] = torch.arange(pa.numel(), dtype=torch.int64, device=dev)
    ra_pairs = pos[_dev(ra_alloc, dev)].cpu().numpy()
    ua_l = [p["ua"] for p in parts if "ua" in p]
    ua = np.sort(pos[_dev(np.concatenate(ua_l), dev)].cpu().numpy()) if ua_l else np.zeros(0, np.int64)
    ut_l = [p["ut"] for p in parts if "ut" in p]
    ut = np.sort(np.concatenate(ut_l)) if ut_l else np.zeros(0, np.int64)
    w_l = [p["warn"] for p in parts if "warn" in p]
    warn = np.sort(np.concatenate(w_l)) if w_l else np.zeros(0, np.int64)
    pa_n, pdl_n = pa.cpu().numpy(), pdl.cpu().numpy()
    u32 = lambda a: np.asarray(a).astype(np.uint32)  # noqa: E731
    return ColumnarFindings(
        n_events=0, dd_offsets=dd_off.astype(np.uint64), dd_members=u32(dd_mem),
        rt_offsets=rt_off.astype(np.uint64), rt_tx=u32(rt_tx), rt_rx=u32(rt_rx), pair_alloc=u32(pa_n),
        pair_delete=np.where(pdl_n < 0, SYN, pdl_n).astype(np.uint32), synthetic_end_ns=int(synth_end),
        warn_index=u32(warn), ra_offsets=ra_off.astype(np.uint64), ra_pairs=u32(ra_pairs), ua_pairs=u32(ua),
        ut_events=u32(ut))


def split(cols: Columns, g: int):
    """Seq-range shards of a trace: [(shard Columns, base index)] for ranks 0..g-1."""
    out = []
    bounds = [cols.n * r // g for r in range(g + 1)]
    for r in range(g):
        a, b = bounds[r], bounds[r + 1]
        sl = slice(a, b)
        out.append((Columns(n=b - a, num_devices_total=cols.num_devices_total, host_device=cols.host_device,
                            seq=cols.seq[sl], start_ns=cols.start_ns[sl], end_ns=cols.end_ns[sl],
                            src_addr=cols.src_addr[sl], dst_addr=cols.dst_addr[sl], bytes=cols.bytes[sl],
                            hash=cols.hash[sl], src_device=cols.src_device[sl], dst_device=cols.dst_device[sl],
                            kind=cols.kind[sl], loc=cols.loc[sl], loc_flags=cols.loc_flags,
                            loc_bucket=cols.loc_bucket, n_buckets=cols.n_buckets, bucket_keys=cols.bucket_keys,
                            wall_time_ns=cols.wall_time_ns, locs=cols.locs), a))
    return out


def run_local(cols: Columns, g: int, strict: bool = False, analyzer: Callable = engine_analyzer):
    """Simulate G ranks as threads (one process, one device): returns rank 0's merged findings."""
    comms = LocalComm.group(g)
    shards = split(cols, g)
    res, errs = [None] * g, [None] * g

    def work(r):
        try:
            res[r] = analyze_sharded(shards[r][0], shards[r][1], comms[r], strict=strict, analyzer=analyzer)
        except BaseException as exc:  # surfaced below
            errs[r] = exc
            comms[r].s.barrier.abort()
    th = [threading.Thread(target=work, args=(r,)) for r in range(g)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    return res[0]


def run_local_device(cols: Columns, g: int, strict: bool = False, device="cuda"):
    """G ranks as threads sharing one device, each with a device-resident shard."""
    from .analysis import DeviceColumns
    comms = LocalComm.group(g)
    shards = [(DeviceColumns(sc, device), b) for sc, b in split(cols, g)]
    res, errs = [None] * g, [None] * g

    def work(r):
        try:
            res[r] = analyze_sharded_device(shards[r][0], shards[r][1], comms[r], strict=strict)
        except BaseException as exc:  # surfaced below
            errs[r] = exc
            comms[r].s.barrier.abort()
    th = [threading.Thread(target=work, args=(r,)) for r in range(g)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    return res[0]
