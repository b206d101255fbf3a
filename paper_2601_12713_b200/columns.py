"""Trace <-> SoA columns: the data format that crosses the C ABI (b2l_trace_cols).

Column layout (one entry per event, event i = trace.events[i]; see DESIGN.md
"Data layout"): seq, start_ns, end_ns, src_addr, dst_addr, bytes, hash as u64;
src_device, dst_device as i32; kind as u8 (0 transfer, 1 alloc, 2 delete,
3 kernel); loc as u32 index into a deduplicated location table.  Per location:
validation flags (model.py:186-190) and the attribution bucket id, i.e. the
dense rank of the report key (0, file, line or 0) / (1, "", codeptr)
(report.py:67-70) -- the only string-typed data, resolved here once per
distinct location instead of once per event.

Values the u64 / i32 columns cannot hold (negative, >= 2**64, non-int) cannot
cross the ABI; ``to_columns`` reports them (``Unrepresentable``) and the
caller produces the reference's violation list for that trace at the boundary.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

U64_MAX = 2**64 - 1
I32_MIN, I32_MAX = -(2**31), 2**31 - 1

LOC_FILE_NO_LINE = 1
LOC_LINE_NONPOS = 2

U64_FIELDS = ("seq", "start_ns", "end_ns", "src_addr", "dst_addr", "bytes", "hash")


class Unrepresentable(ValueError):
    """A field value outside what the device columns can carry."""


@dataclass
class Columns:
    n: int
    num_devices_total: int
    host_device: int
    seq: np.ndarray
    start_ns: np.ndarray
    end_ns: np.ndarray
    src_addr: np.ndarray
    dst_addr: np.ndarray
    bytes: np.ndarray
    hash: np.ndarray
    src_device: np.ndarray
    dst_device: np.ndarray
    kind: np.ndarray
    loc: np.ndarray
    loc_flags: np.ndarray
    loc_bucket: np.ndarray
    n_buckets: int
    bucket_keys: list  # bucket id -> report sort key (report.py:67-70)
    wall_time_ns: Optional[int] = None
    locs: Optional[list] = None  # location id -> (codeptr, file, line)

    @property
    def n_locs(self) -> int:
        return int(self.loc_flags.size)


def _kind_code(kind) -> int:
    v = getattr(kind, "value", kind)
    return {"transfer": 0, "alloc": 1, "delete": 2, "kernel": 3}[v]


def _u64(values, n):
    if n and set(map(type, values)) != {int}:
        raise Unrepresentable("non-int field value")
    try:
        return np.fromiter(values, dtype=np.uint64, count=n)
    except OverflowError as exc:
        raise Unrepresentable(str(exc)) from exc


def _i32(values, n):
    if n and set(map(type, values)) != {int}:
        raise Unrepresentable("non-int device")
    arr = np.fromiter(values, dtype=np.int64, count=n) if n else np.zeros(0, np.int64)
    if n and (arr.min() < I32_MIN or arr.max() > I32_MAX):
        raise Unrepresentable("device number outside int32")
    return arr.astype(np.int32)


def loc_key(codeptr, file, line):
    """report.py:67-70 bucket key."""
    if file is not None:
        return (0, file, line or 0)
    return (1, "", codeptr)


_KIND_CODE = {"transfer": 0, "alloc": 1, "delete": 2, "kernel": 3}
_EV_FIELDS = U64_FIELDS + ("src_device", "dst_device", "kind", "loc")


def to_columns(trace) -> Columns:
    """Convert a Trace (ours or dmlens's) into device-ready columns: one C-level attribute
    sweep per field (operator.attrgetter), locations deduplicated per distinct location object
    first (events usually share them)."""
    from operator import attrgetter
    ev = trace.events
    n = len(ev)
    cols_t = [list(map(attrgetter(f), ev)) for f in _EV_FIELDS]
    cols = {}
    try:
        for k, f in enumerate(U64_FIELDS):
            cols[f] = _u64(cols_t[k], n)
        src = _i32(cols_t[len(U64_FIELDS)], n)
        dst = _i32(cols_t[len(U64_FIELDS) + 1], n)
    except OverflowError as exc:
        raise Unrepresentable(str(exc)) from exc
    kind_of = {}
    for kd in set(cols_t[len(U64_FIELDS) + 2]):
        kind_of[kd] = _KIND_CODE[getattr(kd, "value", kd)]
    kind = np.fromiter(map(kind_of.__getitem__, cols_t[len(U64_FIELDS) + 2]), dtype=np.uint8, count=n)
    # location table: dedupe on (codeptr, file, line); distinct location objects first
    loc_ids: dict = {}
    obj_ids: dict = {}
    flags, bucket_of, locs = [], [], []
    bucket_ids: dict = {}
    bucket_keys = []
    get_loc = attrgetter("codeptr", "file", "line")
    loc_objs = cols_t[len(U64_FIELDS) + 3]
    ids = []
    for loc in loc_objs:
        oid = id(loc)
        lid = obj_ids.get(oid)
        if lid is None:
            k = get_loc(loc)
            lid = loc_ids.get(k)
            if lid is None:
                lid = len(flags)
                loc_ids[k] = lid
                locs.append(k)
                cp, f, ln = k
                fl = 0
                if f is not None and ln is None:
                    fl |= LOC_FILE_NO_LINE
                if ln is not None and ln <= 0:
                    fl |= LOC_LINE_NONPOS
                flags.append(fl)
                bk = loc_key(cp, f, ln)
                bb = bucket_ids.get(bk)
                if bb is None:
                    bb = len(bucket_keys)
                    bucket_ids[bk] = bb
                    bucket_keys.append(bk)
                bucket_of.append(bb)
            obj_ids[oid] = lid
        ids.append(lid)
    loc_arr = np.array(ids, dtype=np.uint32) if n else np.zeros(0, np.uint32)
    return Columns(
        n=n, num_devices_total=int(trace.num_devices_total), host_device=int(trace.host_device),
        seq=cols["seq"], start_ns=cols["start_ns"], end_ns=cols["end_ns"], src_addr=cols["src_addr"],
        dst_addr=cols["dst_addr"], bytes=cols["bytes"], hash=cols["hash"], src_device=src, dst_device=dst,
        kind=kind, loc=loc_arr, loc_flags=np.array(flags, dtype=np.uint8),
        loc_bucket=np.array(bucket_of, dtype=np.uint32), n_buckets=len(bucket_keys), bucket_keys=bucket_keys,
        wall_time_ns=trace.wall_time_ns, locs=locs)


def columns_from_arrays(num_devices_total, host_device, seq, start_ns, end_ns, src_device, dst_device, kind,
                        src_addr, dst_addr, bytes_, hash_, loc=None, loc_flags=None, loc_bucket=None,
                        bucket_keys=None, wall_time_ns=None) -> Columns:
    """Columns straight from numpy arrays (the bench / large-trace path; no Python objects)."""
    n = int(len(seq))
    if loc is None:
        loc = np.zeros(n, dtype=np.uint32)
        loc_flags = np.zeros(1, dtype=np.uint8)
        loc_bucket = np.zeros(1, dtype=np.uint32)
        bucket_keys = [(1, "", 0)]
        locs = [(0, None, None)]
    else:
        locs = None
    return Columns(n=n, num_devices_total=int(num_devices_total), host_device=int(host_device),
                   seq=np.ascontiguousarray(seq, np.uint64), start_ns=np.ascontiguousarray(start_ns, np.uint64),
                   end_ns=np.ascontiguousarray(end_ns, np.uint64), src_addr=np.ascontiguousarray(src_addr, np.uint64),
                   dst_addr=np.ascontiguousarray(dst_addr, np.uint64), bytes=np.ascontiguousarray(bytes_, np.uint64),
                   hash=np.ascontiguousarray(hash_, np.uint64), src_device=np.ascontiguousarray(src_device, np.int32),
                   dst_device=np.ascontiguousarray(dst_device, np.int32), kind=np.ascontiguousarray(kind, np.uint8),
                   loc=np.ascontiguousarray(loc, np.uint32), loc_flags=np.ascontiguousarray(loc_flags, np.uint8),
                   loc_bucket=np.ascontiguousarray(loc_bucket, np.uint32), n_buckets=len(bucket_keys),
                   bucket_keys=list(bucket_keys), wall_time_ns=wall_time_ns, locs=locs)
