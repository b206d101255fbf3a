"""Key-range sharded trace analysis across G ranks.

Input: rank r holds a seq-range shard of the trace (contiguous events
[base_r, base_r + n_r)).  Records go to the rank that owns their key, so that
every detector's state lives on exactly one rank:

  * hash-keyed work -- DD and RT (detectors.py:85-167) only ever relate
    transfers with the same content hash: hashed transfers go to the owner of
    their hash range ((hash * G) >> 64);
  * LIFO pairing (prep.py:45-96) is keyed (dst_device, dst_addr): allocs and
    deletes go to the owner of that key;
  * UT (detectors.py:232-271) relates a target transfer only to the next one
    with the same (device, src_addr) -- given the device's kernel cursor --:
    target transfers go to the owner of (dst_device, src_addr);
  * UA and UT cursors need every kernel of a device (detectors.py:208-212,
    251-253): target kernels are replicated to every rank;
  * RA (detectors.py:170-191) groups pairs by (alloc src_addr, dst_device,
    bytes), a different key from the pairing key: a second exchange sends each
    pair (its alloc and real delete) to the owner of its RA key, where pairing
    is recomputed (a subset of whole LIFO pairs pairs identically) and grouped.

Owners of device-keyed records are the top 32 bits of a splitmix64 mix of the
key times G, >> 32 (route_mix / route_owner here and in b2l_analyze.cu), so a
trace whose work sits on ONE target device (C3) or a few (C4) still spreads
over every rank.  The synthetic-delete time (a trace-wide max, prep.py:61-62)
comes from one all-reduce.  Each rank runs the single-GPU engine on its
sub-traces (a sub-trace keeps global trace order, so every detector is exact
on it); findings then go to rank 0 (one exact-size gather of a flat int64
tensor per rank) and are merged into the reference's global orders (groups by
(first start, key...), pairs by allocation, lists by position), or stay
distributed (gather=False).

The exchange goes through a small communicator interface: ``TorchComm``
(torch.distributed: NCCL on GPUs, gloo on CPU) or ``LocalComm`` (G ranks as
threads of one process -- used to check G-way parity on a single GPU).
"""
from __future__ import annotations

import threading
from typing import Callable, List, Optional

import numpy as np

from .analysis import FLAG_SKIP_ALLOC, FLAG_SKIP_DDRT, FLAG_VALIDATE_ONLY, ColumnarFindings, EngineInvalid

FLAG_NO_VALIDATE = 32  # b2l.h B2L_ANALYZE_NO_VALIDATE: sub-traces of a validated trace (carry kernels repeat a seq)
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

    def allgather_i64(self, a: np.ndarray):
        return [np.asarray(x, np.int64) for x in self._exchange(np.asarray(a, np.int64))]

    def gather0(self, obj):
        out = self._exchange(obj)
        return out if self.rank == 0 else None

    def gatherv_parts(self, t, dst: int = 0):
        """Per-rank tensors -> the list of them on `dst` (None elsewhere)."""
        import torch
        if t.is_cuda:  # another thread's stream reads it next
            torch.cuda.current_stream(t.device).synchronize()
        allp = self._exchange(t)
        return allp if self.rank == dst else None

    def gatherv_parts(self, t, dst: int = 0):
        """Exact-size gather of per-rank tensors (same trailing shape) -> the list of them on
        `dst` (None elsewhere); one size all-gather, then one all_to_all_single in which only
        `dst` receives (NCCL moves device memory; no padding)."""
        torch, dist = self.torch, self.dist
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=self.device)
        ns = [torch.empty_like(n) for _ in range(self.size)]
        dist.all_gather(ns, n)
        sizes = [int(x.item()) for x in ns]
        flat = self.gatherv(t, dst)
        if flat is None:
            return None
        return list(torch.split(flat, sizes))

    def gather0_findings(self, out: dict):
        return self.gather0(out)

    def gather0_findings_dev(self, out: dict):
        import torch
        for v in out.values():  # another thread's stream reads them next
            for t in (v if isinstance(v, tuple) else (v,)):
                if t.is_cuda:
                    torch.cuda.current_stream(t.device).synchronize()
                    break
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

    def allgather_i64(self, a: np.ndarray):
        """Small int64 arrays of any length from every rank (tensor collectives: a size
        all-gather, then one all-gather of max-length buffers)."""
        torch, dist = self.torch, self.dist
        a = np.ascontiguousarray(a, np.int64)
        n = torch.tensor([a.size], dtype=torch.int64, device=self.device)
        ns = [torch.empty_like(n) for _ in range(self.size)]
        dist.all_gather(ns, n)
        sizes = [int(x.item()) for x in ns]
        buf = torch.zeros(max(max(sizes), 1), dtype=torch.int64, device=self.device)
        if a.size:
            buf[:a.size] = torch.from_numpy(a).to(self.device)
        bufs = [torch.empty_like(buf) for _ in range(self.size)]
        dist.all_gather(bufs, buf)
        return [b[:sz].cpu().numpy() for b, sz in zip(bufs, sizes)]

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

    def gatherv_parts(self, t, dst: int = 0):
        """Exact-size gather of per-rank tensors (same trailing shape) -> the list of them on
        `dst` (None elsewhere); one size all-gather, then one all_to_all_single in which only
        `dst` receives (NCCL moves device memory; no padding)."""
        torch, dist = self.torch, self.dist
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=self.device)
        ns = [torch.empty_like(n) for _ in range(self.size)]
        dist.all_gather(ns, n)
        sizes = [int(x.item()) for x in ns]
        flat = self.gatherv(t, dst)
        if flat is None:
            return None
        return list(torch.split(flat, sizes))

    def gather0_findings(self, out: dict):
        """Per-rank findings (dict of numpy arrays / tuples of arrays) to rank 0 as ONE flat int64
        tensor per rank, exact size (gatherv_parts), instead of pickled objects."""
        torch = self.torch
        flat = torch.from_numpy(_pack_findings(out)).to(self.device)
        parts = self.gatherv_parts(flat)
        if parts is None:
            return None
        return [_unpack_findings(p.cpu().numpy()) for p in parts]

    def gather0_findings_dev(self, out: dict):
        """Device findings (dict of device int64 tensors / tuples) to rank 0's device: one flat
        tensor per rank, exact-size gather; unpacked into device tensor views on rank 0."""
        parts = self.gatherv_parts(_pack_findings_dev(out, self.device))
        if parts is None:
            return None
        return [_unpack_findings_dev(p) for p in parts]


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


def _pack_findings_dev(out: dict, dev):
    """_pack_findings for device int64 tensors: the header is built on the host from the tensor
    shapes, the payloads are concatenated on the device (no host round trip)."""
    import torch
    head, body = [], []
    for ki, key in enumerate(_FKEYS):
        if key not in out:
            continue
        val = out[key]
        arrs = val if isinstance(val, tuple) else (val,)
        for slot, t in enumerate(arrs):
            head += [ki, slot if isinstance(val, tuple) else -1, 0, int(t.numel())]
            body.append(t.reshape(-1).to(torch.int64))
    h = torch.tensor([len(head) // 4] + head, dtype=torch.int64, device=body[0].device if body else dev)
    return torch.cat([h] + body)


def _unpack_findings_dev(flat) -> dict:
    nf = int(flat[0].item())
    head = flat[1:1 + 4 * nf].view(nf, 4).cpu().tolist()  # the header only (4 int64 per field)
    o = 1 + 4 * nf
    out: dict = {}
    for ki, slot, _, ln in head:
        seg = flat[o:o + ln]
        o += ln
        key = _FKEYS[ki]
        if slot < 0:
            out[key] = seg
        else:
            out.setdefault(key, []).append(seg)
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


_M64 = (1 << 64) - 1


def route_splitmix(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser over u64 arrays (b2l_analyze.cu route_splitmix)."""
    with np.errstate(over="ignore"):
        z = z.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def route_mix(a, b) -> np.ndarray:
    return route_splitmix(np.asarray(a, np.uint64) ^ route_splitmix(np.asarray(b, np.uint64)))


def route_owner(key: np.ndarray, g: int) -> np.ndarray:
    return (((key >> np.uint64(32)) * np.uint64(g)) >> np.uint64(32)).astype(np.int64)


def _u32dev(d) -> np.ndarray:
    """A device column as the kernels read it in a key: (uint64_t)(uint32_t)dst."""
    return np.asarray(d).astype(np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)


def device_owners(cols: Columns, g: int):
    """Owners of the device-keyed records: (alloc/delete mask, owner), (target-transfer mask,
    owner).  Pairing keys (dst_device, dst_addr) go to (dst_device + owner(mix(dst_addr))) % g:
    traces that reuse one device address per device (C2/C5 cycles) still put each device on its
    own rank, and many addresses per device spread further.  UT keys (dst_device, src_addr) go to
    owner(mix(dst_device ^ 2^40, src_addr))."""
    kind, dst = cols.kind, cols.dst_device.astype(np.int64)
    host = cols.host_device
    ad = (kind == ALLOC) | (kind == DELETE)
    tt = (kind == TRANSFER) & (dst != host)
    du = _u32dev(dst)
    o_ad = (du.astype(np.int64) + route_owner(route_splitmix(np.asarray(cols.dst_addr, np.uint64)), g)) % g
    o_tt = route_owner(route_mix(du ^ np.uint64(1 << 40), cols.src_addr), g)
    return (ad, o_ad), (tt, o_tt)


def kernel_summary(cols: Columns):
    """Per target device of a shard: (has kernels, max kernel end) -- all-gathered, they give
    every rank the carry (max end of the device's kernels on earlier ranks)."""
    nd = cols.num_devices_total
    tk = (cols.kind == KERNEL) & (cols.dst_device.astype(np.int64) != cols.host_device)
    d = cols.dst_device[tk].astype(np.int64)
    has = np.bincount(d, minlength=nd)[:nd] > 0
    mx = np.zeros(nd, np.uint64)
    np.maximum.at(mx, d, cols.end_ns[tk].astype(np.uint64))
    return has, mx


def kernel_carry(all_has, all_max, rank):
    """(has carry, carry end) per device for `rank`: the max end of the device's kernels on the
    ranks before it (UA / UT cursors that land there, detectors.py:208-212,251-253)."""
    nd = all_has.shape[1]
    has = np.zeros(nd, bool)
    mx = np.zeros(nd, np.uint64)
    for q in range(rank):
        has |= all_has[q]
        mx = np.where(all_has[q], np.maximum(mx, all_max[q]), mx)
    return has, mx


def cursor_kernels(cols: Columns, q_idx: np.ndarray, carry_has, carry_max) -> np.ndarray:
    """For each query event (a target transfer or alloc), the LOCAL kernel its cursor lands on
    (the first kernel of its device, in trace order, whose prefix-max end reaches the query's
    start: detectors.py:208-212 / 251-253), or -1 when the cursor lands on an earlier rank's
    kernel (carry >= start) or a later rank's (no local kernel reaches it)."""
    host = cols.host_device
    tk = np.nonzero((cols.kind == KERNEL) & (cols.dst_device.astype(np.int64) != host))[0]
    kd = cols.dst_device[tk].astype(np.int64)
    out = np.full(q_idx.size, -1, np.int64)
    qd = cols.dst_device[q_idx].astype(np.int64)
    qt = cols.start_ns[q_idx].astype(np.uint64)
    for d in np.unique(qd):
        K = tk[kd == d]
        sel = np.nonzero(qd == d)[0]
        if K.size == 0:
            continue
        pm = np.maximum.accumulate(cols.end_ns[K].astype(np.uint64))
        c = np.searchsorted(pm, qt[sel], side="left")
        ok = c < K.size
        if carry_has[d]:
            ok &= ~(carry_max[d] >= qt[sel])
        out[sel[ok]] = K[c[ok]]
    return out


def ra_owner(src_addr, dst_device, nbytes, g: int) -> np.ndarray:
    """Owner of a pair's RA key (alloc src_addr, dst_device, bytes)."""
    return route_owner(route_mix(src_addr, route_mix(_u32dev(dst_device), nbytes)), g)


def device_parts(shard: Columns, base: int, G: int, ad_o, tt_o, c_has, c_max):
    """Space-1 rows of a seq-range shard for every rank, each in trace order: allocs/deletes to
    their pairing owner, target transfers to their UT owner, and the kernels those ranks need for
    exact UA / UT cursors without replicating every kernel: each query's local cursor kernel (to
    the query's rank, once), the shard's first kernel of every device (to every rank: the cursor
    of a query whose kernel lies on a later rank), and per device a carry kernel (end = the max
    kernel end on earlier ranks, start = the shard's first start; to every rank, ahead of the
    shard's rows) standing in for a cursor that lands on an earlier rank.  Kernels in a rank's
    sub-trace are then a subset of the trace's kernels (plus carry kernels whose end never
    exceeds the true prefix max before them), which leaves every cursor where the whole trace
    puts it."""
    (ad, o_ad), (tt, o_tt) = ad_o, tt_o
    n = shard.n
    host = shard.host_device
    dst = shard.dst_device.astype(np.int64)
    q_alloc = ad & (shard.kind == ALLOC) & (dst != host)
    q_idx = np.nonzero(q_alloc | tt)[0]
    q_own = np.where(tt[q_idx], o_tt[q_idx], o_ad[q_idx])
    cur = cursor_kernels(shard, q_idx, c_has, c_max) if q_idx.size else np.zeros(0, np.int64)
    tk = np.nonzero((shard.kind == KERNEL) & (dst != host))[0]
    first_k = tk[np.unique(dst[tk], return_index=True)[1]] if tk.size else np.zeros(0, np.int64)
    first_start = int(shard.start_ns[0]) if n else 0
    out = []
    for r in range(G):
        sel = np.zeros(n, bool)
        sel |= ad & (o_ad == r)
        sel |= tt & (o_tt == r)
        sel[cur[(q_own == r) & (cur >= 0)]] = True
        sel[first_k] = True
        rows = _rows(shard, np.nonzero(sel)[0], base)
        carry_d = [d for d in range(c_has.size) if c_has[d] and int(c_max[d]) >= first_start and n]
        if carry_d:
            pr = np.zeros((len(carry_d), ROW), np.uint64)
            pr[:, 0] = base
            pr[:, 1] = shard.seq[0]
            pr[:, 2] = first_start
            pr[:, 3] = c_max[carry_d]
            pr[:, 8] = np.asarray(carry_d, np.uint64)
            pr[:, 9] = np.asarray(carry_d, np.uint64)
            pr[:, 10] = KERNEL
            pr[:, 11] = shard.loc[0]
            rows = np.concatenate([pr, rows])
        out.append(rows)
    return out


def _rows_gid(cols: Columns, idx: np.ndarray, gid: np.ndarray) -> np.ndarray:
    r = _rows(cols, idx, 0)
    r[:, 0] = np.asarray(gid, np.int64)[idx].astype(np.uint64)
    return r


def _tag(rows: np.ndarray, space: int) -> np.ndarray:
    rows = rows.copy()
    rows[:, 0] |= np.uint64(space) << np.uint64(63)
    return rows


def _receive(got):
    rec = np.concatenate(got) if got else np.zeros((0, ROW), np.uint64)
    space = rec[:, 0] >> np.uint64(63)
    rec = rec.copy()
    rec[:, 0] &= np.uint64((1 << 63) - 1)
    return rec, space


# ------------------------------------------------------------------------ the sharded pipeline
def engine_analyzer(cols, flags=0, synthetic_end_ns=None, strict=False):
    from .analysis import analyze_columns
    return analyze_columns(cols, strict=strict, flags=flags, synthetic_end_ns=synthetic_end_ns)


def _boundary_check(comm, first, last, bad_i, bad_r, base):
    """The order rule across shard boundaries (model.py:193-196) from every rank's edge events,
    and the global violation list.  One all-gather of 5 int64 per rank, then (only when a rank
    found violations) one exact-size all-gather of the flagged indices."""
    G = comm.size
    edge = np.array([1, first[0], first[1], last[0], last[1]] if first is not None else [0, 0, 0, 0, 0],
                    np.uint64).view(np.int64)
    edges = [e.view(np.uint64) for e in comm.allgather_i64(edge)]
    prev = None
    for r in range(comm.rank):
        if int(edges[r][0]):
            prev = edges[r]
    if prev is not None and first is not None:
        s0, q0 = first
        m = 0
        if s0 < int(prev[3]) or (s0 == int(prev[3]) and q0 < int(prev[4])):
            m |= 1 << 10
        if q0 <= int(prev[4]):
            m |= 1 << 11
        if m:
            k = np.nonzero(bad_i == 0)[0]
            if k.size:
                bad_r[k[0]] |= m
            else:
                bad_i, bad_r = np.concatenate([[0], bad_i]), np.concatenate([[m], bad_r]).astype(np.uint32)
    nbad = comm.allgather_i64(np.array([bad_i.size], np.int64))
    if sum(int(x[0]) for x in nbad) == 0:
        return
    mine = np.concatenate([(bad_i + base).astype(np.int64), bad_r.astype(np.int64)])
    allb = comm.allgather_i64(mine)
    gi = np.concatenate([a[:a.size // 2] for a in allb])
    gr = np.concatenate([a[a.size // 2:] for a in allb])
    raise EngineInvalid(gi.astype(np.uint32), gr.astype(np.uint32))


def _findings_h(f, sub, gid):
    """DD/RT findings of a hash sub-trace (host columns), global indices + group sort keys."""
    out = {}
    off = f.dd_offsets.astype(np.int64)
    mem = f.dd_members.astype(np.int64)
    fl = mem[off[:-1]] if off.size > 1 else np.zeros(0, np.int64)
    out["dd"] = (off, gid[mem], sub.start_ns[fl], sub.hash[fl], sub.dst_device[fl], gid[fl])
    off = f.rt_offsets.astype(np.int64)
    tx, rx = f.rt_tx.astype(np.int64), f.rt_rx.astype(np.int64)
    ft = tx[off[:-1]] if off.size > 1 else np.zeros(0, np.int64)
    out["rt"] = (off, gid[tx], gid[rx], sub.start_ns[ft], sub.hash[ft], sub.src_device[ft], sub.dst_device[ft])
    return out


def _findings_d(f, gid):
    """pairs, warnings, UA, UT of a device sub-trace (run 1), global indices."""
    pa = f.pair_alloc.astype(np.int64)
    pd = f.pair_delete
    return {"pairs": (gid[pa], np.where(pd == SYN, -1, gid[np.where(pd == SYN, 0, pd).astype(np.int64)])),
            "warn": gid[f.warn_index.astype(np.int64)], "ua": gid[pa[f.ua_pairs.astype(np.int64)]],
            "ut": gid[f.ut_events.astype(np.int64)]}


def _findings_ra(f, sub, gid):
    """RA groups of an RA sub-trace (run 2): alloc global indices + group sort keys."""
    pa = f.pair_alloc.astype(np.int64)
    off = f.ra_offsets.astype(np.int64)
    fa = pa[f.ra_pairs[off[:-1]].astype(np.int64)] if off.size > 1 else np.zeros(0, np.int64)
    return {"ra": (off, gid[pa[f.ra_pairs.astype(np.int64)]], sub.start_ns[fa], sub.src_addr[fa], sub.dst_device[fa],
                   sub.bytes[fa])}


def analyze_sharded(shard: Columns, base: int, comm, strict: bool = False,
                    analyzer: Callable = engine_analyzer) -> Optional[ColumnarFindings]:
    """Findings of the whole trace (global event indices) on rank 0, None elsewhere (host
    columns; the exchange moves host rows).  Raises EngineInvalid (global indices) on every rank
    if any shard fails validation."""
    G = comm.size
    # ---- 1. validation of every shard + the order rule across shard boundaries (model.py:193-196)
    bad_i, bad_r = np.zeros(0, np.int64), np.zeros(0, np.uint32)
    try:
        analyzer(shard, flags=FLAG_VALIDATE_ONLY)
    except EngineInvalid as exc:
        bad_i, bad_r = exc.bad_index.astype(np.int64), exc.bad_rules.astype(np.uint32)
    n = shard.n
    _boundary_check(comm, (int(shard.start_ns[0]), int(shard.seq[0])) if n else None,
                    (int(shard.start_ns[-1]), int(shard.seq[-1])) if n else None, bad_i, bad_r, base)

    # ---- 2. one all-to-all: hashed transfers by hash range, device work by device key
    kind, nb, h = shard.kind, shard.bytes, shard.hash
    is_h = (kind == TRANSFER) & (nb > 0) & (h != 0)
    (ad, o_ad), (tt, o_tt) = device_owners(shard, G)
    dmax = int(shard.end_ns[kind != KERNEL].max()) if np.any(kind != KERNEL) else 0
    has, mx = kernel_summary(shard)
    allk = comm.allgather_i64(np.concatenate([has.astype(np.int64), mx.view(np.int64)]))
    nd = has.size
    all_has = np.stack([a[:nd] > 0 for a in allk])
    all_max = np.stack([a[nd:].view(np.uint64) for a in allk])
    c_has, c_max = kernel_carry(all_has, all_max, comm.rank)
    parts_d = device_parts(shard, base, G, (ad, o_ad), (tt, o_tt), c_has, c_max)
    ih = np.nonzero(is_h)[0]
    oh = hash_owner(h[ih], G)
    rows_h = _rows(shard, ih, base)
    parts = [np.concatenate([_tag(rows_h[oh == r], 0), _tag(parts_d[r], 1)]) for r in range(G)]
    rec, space = _receive(comm.alltoall(parts))
    synth_end = comm.allreduce_max(dmax)
    sub_h, gid_h = _subtrace(rec[space == 0], shard)
    sub_d, gid_d = _subtrace(rec[space == 1], shard)

    # ---- 3. per-rank engine runs: DD/RT on the hash sub-trace; pairs, UA, UT on the device one
    out = {}
    if sub_h.n:
        out.update(_findings_h(analyzer(sub_h, flags=FLAG_SKIP_ALLOC, strict=strict), sub_h, gid_h))
    f = analyzer(sub_d, flags=FLAG_SKIP_DDRT | FLAG_NO_VALIDATE, synthetic_end_ns=synth_end) if sub_d.n else None
    if f is not None:
        out.update(_findings_d(f, gid_d))

    # ---- 4. second exchange: whole pairs to the owner of their RA key; pairing + RA there
    parts = [np.zeros((0, ROW), np.uint64) for _ in range(G)]
    if f is not None and f.pair_alloc.size:
        pa = f.pair_alloc.astype(np.int64)
        pd = f.pair_delete
        real = pd != SYN
        o = ra_owner(sub_d.src_addr[pa], sub_d.dst_device[pa], sub_d.bytes[pa], G)
        dest = np.full(sub_d.n, -1, np.int64)
        dest[pa] = o
        dest[pd[real].astype(np.int64)] = o[real]
        parts = [_tag(_rows_gid(sub_d, np.nonzero(dest == r)[0], gid_d), 1) for r in range(G)]
    rec, _ = _receive(comm.alltoall(parts))
    sub_r, gid_r = _subtrace(rec, shard)
    if sub_r.n:
        out.update(_findings_ra(analyzer(sub_r, flags=FLAG_SKIP_DDRT | FLAG_NO_VALIDATE, synthetic_end_ns=synth_end),
                                sub_r, gid_r))
    parts = comm.gather0_findings(out)
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
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p]
    L.b2l_shard_kernel_summary.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    L.b2l_shard_route_pairs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]
    L.b2l_shard_unpack.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                   ctypes.c_void_p]
    return L, _lib


def _torch_done(dev):
    """The engine runs on its own streams: device tensors torch just wrote (uploads, the received
    rows, gathers) must be complete before a b2l call reads them."""
    import torch
    if dev.type == "cuda":
        torch.cuda.current_stream(dev).synchronize()


def _kernel_summary_dev(shard):
    """b2l_shard_kernel_summary: (has target kernels, max target-kernel end) per device."""
    import ctypes
    L, _lib = _shard_lib()
    nd = shard.host.num_devices_total
    _torch_done(shard.t["seq"].device)
    has, mx = np.zeros(nd, np.uint64), np.zeros(nd, np.uint64)
    _lib.check(L.b2l_shard_kernel_summary(ctypes.addressof(shard.struct), has.ctypes.data, mx.ctypes.data),
               "b2l_shard_kernel_summary")
    return has > 0, mx


def _route(shard, base: int, G: int, c_has, c_max):
    """b2l_shard_route: device rows grouped by destination rank, counts, max data-op end (a
    sizing call for an upper bound of the rows, then the routing call)."""
    import ctypes

    import torch
    L, _lib = _shard_lib()
    dev = shard.t["seq"].device
    _torch_done(dev)
    counts = np.zeros(G, np.uint64)
    nrec, dend = ctypes.c_uint64(0), ctypes.c_uint64(0)
    ch = np.ascontiguousarray(c_has, np.uint8)
    cm = np.ascontiguousarray(c_max, np.uint64)
    args = (ctypes.addressof(shard.struct), G, base, 0, ch.ctypes.data, cm.ctypes.data)
    _lib.check(L.b2l_shard_route(*args, None, counts.ctypes.data, ctypes.addressof(nrec), ctypes.addressof(dend)),
               "b2l_shard_route")
    rows = torch.empty((max(nrec.value, 1), ROW), dtype=torch.int64, device=dev)
    if nrec.value:
        _lib.check(L.b2l_shard_route(*args, rows.data_ptr(), counts.ctypes.data, ctypes.addressof(nrec),
                                     ctypes.addressof(dend)), "b2l_shard_route")
    return rows[:int(counts.sum())], counts, int(dend.value)


def _route_pairs(sub, gid, f, G: int):
    """b2l_shard_route_pairs: whole pairs of a device sub-trace to the owners of their RA keys."""
    import ctypes

    import torch
    L, _lib = _shard_lib()
    dev = gid.device
    counts = np.zeros(G, np.uint64)
    if f is None or f.pair_alloc.size == 0:
        return torch.empty((0, ROW), dtype=torch.int64, device=dev), counts
    pa = torch.from_numpy(np.ascontiguousarray(f.pair_alloc, np.uint32).view(np.int32)).to(dev)
    pd = torch.from_numpy(np.ascontiguousarray(f.pair_delete, np.uint32).view(np.int32)).to(dev)
    _torch_done(dev)
    nrec = ctypes.c_uint64(0)
    args = (ctypes.addressof(sub.struct), gid.data_ptr(), pa.data_ptr(), pd.data_ptr(), pa.numel(), G)
    _lib.check(L.b2l_shard_route_pairs(*args, None, counts.ctypes.data, ctypes.addressof(nrec)),
               "b2l_shard_route_pairs")
    rows = torch.empty((max(nrec.value, 1), ROW), dtype=torch.int64, device=dev)
    if nrec.value:
        _lib.check(L.b2l_shard_route_pairs(*args, rows.data_ptr(), counts.ctypes.data, ctypes.addressof(nrec)),
                   "b2l_shard_route_pairs")
    return rows[:nrec.value], counts


def _unpack(recv, space: int, like):
    """Rows of one key space -> (DeviceColumns sub-trace, global indices as a device tensor)."""
    import ctypes

    import torch

    from .analysis import DeviceColumns
    L, _lib = _shard_lib()
    m, dev = recv.shape[0], recv.device
    _torch_done(dev)
    dt = {"src_device": torch.int32, "dst_device": torch.int32, "kind": torch.uint8, "loc": torch.int32}
    t = {f: torch.empty(max(m, 1), dtype=dt.get(f, torch.int64), device=dev) for f in _SHARD_FIELDS}
    ptrs = (ctypes.c_void_p * len(_SHARD_FIELDS))(*[t[f].data_ptr() for f in _SHARD_FIELDS])
    n = ctypes.c_uint64(0)
    _lib.check(L.b2l_shard_unpack(recv.data_ptr() if m else None, m, space, ptrs, ctypes.addressof(n)),
               "b2l_shard_unpack")
    k = n.value
    gid = t.pop("gid")[:k]
    return DeviceColumns.from_device({f: v[:k] for f, v in t.items()}, k, like), gid


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


def _ix(a, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(dev)


def _findings_h_dev(f, sub, gid):
    """_findings_h on device tensors (global indices and sort keys gathered on the device)."""
    dev, t = gid.device, sub.t
    off, mem = _ix(f.dd_offsets.astype(np.int64), dev), _ix(f.dd_members, dev)
    fl = mem[off[:-1]]
    out = {"dd": (off, gid[mem], t["start_ns"][fl], t["hash"][fl], t["dst_device"][fl].long(), gid[fl])}
    off, tx, rx = _ix(f.rt_offsets.astype(np.int64), dev), _ix(f.rt_tx, dev), _ix(f.rt_rx, dev)
    ft = tx[off[:-1]]
    out["rt"] = (off, gid[tx], gid[rx], t["start_ns"][ft], t["hash"][ft], t["src_device"][ft].long(),
                 t["dst_device"][ft].long())
    return out


def _findings_d_dev(f, gid):
    import torch
    dev = gid.device
    pa = _ix(f.pair_alloc, dev)
    pd = _ix(f.pair_delete, dev)
    syn = pd == int(SYN)
    return {"pairs": (gid[pa], torch.where(syn, torch.full_like(pd, -1), gid[torch.where(syn, 0, pd)])),
            "warn": gid[_ix(f.warn_index, dev)], "ua": gid[pa[_ix(f.ua_pairs, dev)]], "ut": gid[_ix(f.ut_events, dev)]}


def _findings_ra_dev(f, sub, gid):
    dev, t = gid.device, sub.t
    pa = _ix(f.pair_alloc, dev)
    off = _ix(f.ra_offsets.astype(np.int64), dev)
    rp = _ix(f.ra_pairs, dev)
    fa = pa[rp[off[:-1]]]
    return {"ra": (off, gid[pa[rp]], t["start_ns"][fa], t["src_addr"][fa], t["dst_device"][fa].long(), t["bytes"][fa])}


def analyze_sharded_device(shard, base: int, comm, strict: bool = False, gather: bool = True):
    """The sharded pipeline with every event-sized step on the device: ``shard`` is a
    DeviceColumns seq-range shard; validation, routing (b2l_shard_route), the all-to-all of
    the rows (NCCL on device memory), unpacking (b2l_shard_unpack), the engine runs, the RA
    exchange (b2l_shard_route_pairs) and the findings (global indices and group sort keys as
    device tensors) stay in HBM; the gather moves them to rank 0's device, where they are merged.
    Same results and exceptions as ``analyze_sharded``.  ``gather=False`` stops before the gather:
    every rank returns its own key ranges' findings (device tensors, global indices)."""
    import torch

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
    n = host.n
    _boundary_check(comm, (int(host.start_ns[0]), int(host.seq[0])) if n else None,
                    (int(host.start_ns[-1]), int(host.seq[-1])) if n else None, bad_i, bad_r, base)
    ph.mark("validate")
    # ---- 2. kernel carries (one tiny all-gather), route + one all-to-all of device rows
    has, mx = _kernel_summary_dev(shard)
    nd = has.size
    allk = comm.allgather_i64(np.concatenate([has.astype(np.int64), mx.view(np.int64)]))
    c_has, c_max = kernel_carry(np.stack([a[:nd] > 0 for a in allk]), np.stack([a[nd:].view(np.uint64) for a in allk]),
                                comm.rank)
    if n:
        rows, counts, dmax = _route(shard, base, G, c_has, c_max)
    else:
        rows, counts, dmax = torch.empty((0, ROW), dtype=torch.int64, device=shard.t["seq"].device), \
            np.zeros(G, np.uint64), 0
    ph.mark("route")
    recv = comm.alltoall_rows(rows, counts)
    synth_end = comm.allreduce_max(dmax)
    ph.mark("exchange")
    sub_h, gid_h = _unpack(recv, 0, shard)
    sub_d, gid_d = _unpack(recv, 1, shard)
    ph.mark("unpack")
    # ---- 3. per-rank engine runs on the device sub-traces
    out = {}
    if sub_h.n:
        out.update(_findings_h_dev(analyzer_dev(sub_h, flags=FLAG_SKIP_ALLOC, strict=strict), sub_h, gid_h))
    f = analyzer_dev(sub_d, flags=FLAG_SKIP_DDRT | FLAG_NO_VALIDATE, synthetic_end_ns=synth_end) if sub_d.n else None
    if f is not None:
        out.update(_findings_d_dev(f, gid_d))
    ph.mark("engine")
    # ---- 4. second exchange: whole pairs to the owners of their RA keys; RA there
    rows2, counts2 = _route_pairs(sub_d, gid_d, f, G)
    recv2 = comm.alltoall_rows(rows2, counts2)
    if recv2.shape[0] > 1:  # each source's rows are in global order, the sources' ranges interleave
        recv2 = recv2[_sort_pairs_dev(torch.zeros_like(recv2[:, 0]), recv2[:, 0] & ((1 << 63) - 1))]
    sub_r, gid_r = _unpack(recv2, 1, shard)
    if sub_r.n:
        out.update(_findings_ra_dev(analyzer_dev(sub_r, flags=FLAG_SKIP_DDRT | FLAG_NO_VALIDATE,
                                                 synthetic_end_ns=synth_end), sub_r, gid_r))
    ph.mark("ra")
    if not gather:
        return out
    parts = comm.gather0_findings_dev(out)
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
def _sort_pairs_dev(k0, k1):
    """Stable order of (k0, k1) u64 key pairs on the device (b2l_sort_u64_pairs_device: LSD radix
    over the live bytes)."""
    import ctypes

    import torch

    from . import _lib
    L = _lib.lib()
    L.b2l_sort_u64_pairs_device.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    n = k0.numel()
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=k0.device)
    if n < 2:
        return torch.arange(n, dtype=torch.int64, device=k0.device)
    a, b = k0.contiguous(), k1.contiguous()
    torch.cuda.current_stream(k0.device).synchronize()  # the sort runs on the engine's stream
    _lib.check(L.b2l_sort_u64_pairs_device(a.data_ptr(), b.data_ptr(), n, perm.data_ptr()),
               "b2l_sort_u64_pairs_device")
    return perm[:n].long()


def _dev_lexsort(kcols, dev):
    """Order of u64 key columns (first = primary): LSD passes of the stable pair sort, (k[-2],
    k[-1]) first, then (k[-4], k[-3])."""
    import torch
    n = kcols[0].numel()
    order = torch.arange(n, dtype=torch.int64, device=dev)
    if n < 2:
        return order
    cols = list(kcols)
    if len(cols) % 2:
        cols = [torch.zeros(n, dtype=torch.int64, device=dev)] + cols
    for j in range(len(cols) - 2, -1, -2):
        order = order[_sort_pairs_dev(cols[j][order], cols[j + 1][order])]
    return order


def _merge_groups_dev(parts, key, member_cols, sort_cols, dev):
    """_merge_groups on device tensors: one engine sort for the group order, the member ranges
    gathered with a repeat/arange index."""
    import torch
    ps = [p[key] for p in parts if key in p]
    if not ps or sum(int(t[0].numel()) - 1 for t in ps) == 0:
        return torch.zeros(1, dtype=torch.int64, device=dev), [torch.zeros(0, dtype=torch.int64, device=dev)
                                                                for _ in member_cols]
    sizes = torch.cat([t[0][1:] - t[0][:-1] for t in ps])
    base, bases = 0, []
    for t in ps:
        bases.append(t[0][:-1] + base)
        base += int(t[1].numel())
    starts = torch.cat(bases)
    keys = [torch.cat([t[c] for t in ps]) for c in sort_cols]
    order = _dev_lexsort(keys, dev)
    sz, st = sizes[order], starts[order]
    first = torch.cumsum(sz, 0) - sz
    total = base
    idx = torch.repeat_interleave(st - first, sz, output_size=total) + torch.arange(total, device=dev)
    new_off = torch.zeros(sizes.numel() + 1, dtype=torch.int64, device=dev)
    new_off[1:] = torch.cumsum(sz, 0)
    flat = [torch.cat([t[c] for t in ps])[idx] for c in member_cols]
    return new_off, flat


def _merge_dev(parts, synth_end, dev) -> ColumnarFindings:
    """_merge on rank 0's GPU from device tensors: group orders by the engine's radix sort, index
    work as device gathers; one copy of the merged findings to the host at the end."""
    import torch
    z = torch.zeros(0, dtype=torch.int64, device=dev)
    cat = lambda key, k: torch.cat([p[key][k] if isinstance(p[key], tuple) else p[key]  # noqa: E731
                                    for p in parts if key in p]) if any(key in p for p in parts) else z
    dd_off, (dd_mem,) = _merge_groups_dev(parts, "dd", [1], [2, 3, 4], dev)
    rt_off, (rt_tx, rt_rx) = _merge_groups_dev(parts, "rt", [1, 2], [3, 4, 5, 6], dev)
    pa, pdl = cat("pairs", 0), cat("pairs", 1)
    o = _sort_pairs_dev(torch.zeros_like(pa), pa) if pa.numel() > 1 else torch.arange(pa.numel(), device=dev)
    pa, pdl = pa[o], pdl[o]
    ra_off, (ra_alloc,) = _merge_groups_dev(parts, "ra", [1], [2, 3, 4, 5], dev)
    pos = torch.zeros(int(pa.max().item()) + 1 if pa.numel() else 1, dtype=torch.int64, device=dev)
    pos[pa] = torch.arange(pa.numel(), dtype=torch.int64, device=dev)
    ra_pairs = pos[ra_alloc]
    ua = torch.sort(pos[cat("ua", 0)]).values
    ut = torch.sort(cat("ut", 0)).values
    warn = torch.sort(cat("warn", 0)).values
    h = lambda t: t.cpu().numpy()  # noqa: E731
    u32 = lambda t: h(t).astype(np.uint32)  # noqa: E731
    pdl_n = h(pdl)
    return ColumnarFindings(
        n_events=0, dd_offsets=h(dd_off).astype(np.uint64), dd_members=u32(dd_mem),
        rt_offsets=h(rt_off).astype(np.uint64), rt_tx=u32(rt_tx), rt_rx=u32(rt_rx), pair_alloc=u32(pa),
        pair_delete=np.where(pdl_n < 0, SYN, pdl_n).astype(np.uint32), synthetic_end_ns=int(synth_end),
        warn_index=u32(warn), ra_offsets=h(ra_off).astype(np.uint64), ra_pairs=u32(ra_pairs), ua_pairs=u32(ua),
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
