"""Standalone detector entry points -- drop-ins for the reference's public helpers.

  validate(trace)                                           model.py:125-200
  get_alloc_delete_pairs(data_op_events, warn)              prep.py:45-96
  sort_by_device(events, num_devices_total, key)            prep.py:99-115
  find_duplicate_transfers(data_op_events)                  detectors.py:85-103
  find_round_trips(data_op_events, strict_pseudocode)       detectors.py:106-167
  find_repeated_allocs(data_op_events, warn)                detectors.py:184-191
  find_unused_allocs(tgt_events, data_op_events, ndev, warn) detectors.py:219-229
  find_unused_transfers(tgt_events, data_op_events, ndev)   detectors.py:232-271

Like the reference, these take event lists as given (no validation, no kind
filtering beyond what each function itself does; lists in chronological order
as the reference requires).  Each list is turned into a pseudo-trace whose rows
carry the role the function gives them -- e.g. every row of
find_duplicate_transfers is a hashed transfer, every tgt_event of the unused
detectors is a kernel interval on its dst device, and no device is the host --
and the same CUDA pipeline as analyze() runs on it (b2l_analyze_ex with
NO_VALIDATE / RAW_HASHED / SKIP_* flags).  Results reference the caller's
objects.
"""
from __future__ import annotations

import ctypes
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from .analysis import (FLAG_SKIP_ALLOC, FLAG_SKIP_DDRT, FLAG_VALIDATE_ONLY, SYNTHETIC, WARN_REASON, EngineInvalid,
                       _boundary_violations, _event_violations, _header_violations, analyze_columns)
from .columns import Columns, Unrepresentable, to_columns
from .errors import DeviceOutOfRange as _OwnDeviceOutOfRange
from .types import type_family

FLAG_NO_VALIDATE, FLAG_RAW_HASHED = 32, 64
TRANSFER, ALLOC, DELETE, KERNEL = 0, 1, 2, 3
_KIND = {"transfer": TRANSFER, "alloc": ALLOC, "delete": DELETE, "kernel": KERNEL}


def _family(events):
    return type_family(events[0]) if events else type_family(object())


def _kind(e):
    return _KIND[getattr(e.kind, "value", e.kind)]


def _pseudo(rows, ndev):
    """rows: list of (event, kind_code) in row order -> Columns with host = -1."""
    n = len(rows)
    U = lambda f: np.fromiter((getattr(e, f) for e, _ in rows), dtype=np.uint64, count=n)  # noqa: E731
    I = lambda f: np.fromiter((getattr(e, f) for e, _ in rows), dtype=np.int64, count=n).astype(np.int32)  # noqa
    return Columns(n=n, num_devices_total=int(ndev), host_device=-1, seq=U("seq"), start_ns=U("start_ns"),
                   end_ns=U("end_ns"), src_addr=U("src_addr"), dst_addr=U("dst_addr"), bytes=U("bytes"),
                   hash=U("hash"), src_device=I("src_device"), dst_device=I("dst_device"),
                   kind=np.fromiter((k for _, k in rows), dtype=np.uint8, count=n),
                   loc=np.zeros(n, np.uint32), loc_flags=np.zeros(1, np.uint8), loc_bucket=np.zeros(1, np.uint32),
                   n_buckets=1, bucket_keys=[(1, "", 0)], wall_time_ns=None, locs=[(0, None, None)])


def _ndev_of(events):
    if not events:
        return 1
    return max(max(e.src_device for e in events), max(e.dst_device for e in events)) + 1


# ------------------------------------------------------------------------ validate (model.py:125-200)
def validate(trace):
    T = type_family(trace)
    try:
        cols = to_columns(trace)
    except Unrepresentable:
        return _boundary_violations(trace, T.Violation)
    head = _header_violations(trace, T.Violation)
    try:
        analyze_columns(cols, flags=FLAG_VALIDATE_ONLY)
    except EngineInvalid as exc:
        return head + _event_violations(trace, exc.bad_index, exc.bad_rules, T.Violation)
    return head


# ------------------------------------------------------------------------ pairs (prep.py)
def _pairs_from(data_op_events, T, warn, extra_rows=(), ndev=None, flags=FLAG_SKIP_DDRT):
    rows = [(e, _kind(e) if _kind(e) in (ALLOC, DELETE) else TRANSFER) for e in data_op_events]
    rows += list(extra_rows)
    order = np.argsort(np.fromiter((e.start_ns for e, _ in rows), dtype=np.uint64, count=len(rows)),
                       kind="stable") if extra_rows else np.arange(len(rows))
    rows_sorted = [rows[i] for i in order]
    cols = _pseudo(rows_sorted, ndev if ndev is not None else _ndev_of([e for e, _ in rows]))
    cf = analyze_columns(cols, flags=FLAG_NO_VALIDATE | flags)
    ev = [e for e, _ in rows_sorted]
    if warn is not None:
        for i in cf.warn_index.tolist():
            warn(T.PrepWarning(ev[i].seq, WARN_REASON))
    pairs = []
    end = cf.synthetic_end_ns
    for a, d in zip(cf.pair_alloc.tolist(), cf.pair_delete.tolist()):
        al = ev[a]
        if d == SYNTHETIC:
            syn = T.TraceEvent(seq=al.seq, kind=T.EventKind.DELETE, start_ns=end, end_ns=end,
                               src_device=al.src_device, dst_device=al.dst_device, src_addr=0, dst_addr=al.dst_addr,
                               bytes=0, hash=0, loc=al.loc)
            pairs.append(T.AllocPair(al, syn, synthetic_delete=True))
        else:
            pairs.append(T.AllocPair(al, ev[d]))
    return cf, ev, pairs


def get_alloc_delete_pairs(data_op_events: Sequence, warn: Optional[Callable] = None):
    if not data_op_events:
        return []
    T = _family(data_op_events)
    return _pairs_from(list(data_op_events), T, warn)[2]


def _device_error(events):
    if events and type(events[0]).__module__.startswith("dmlens"):
        import importlib
        return importlib.import_module(type(events[0]).__module__.split(".")[0] + ".prep").DeviceOutOfRange
    return _OwnDeviceOutOfRange


def sort_by_device(events: Sequence, num_devices_total: int, key: str = "dst"):
    if key not in ("src", "dst"):
        raise ValueError(f"key must be 'src' or 'dst', got {key!r}")
    events = list(events)
    devs = [e.src_device if key == "src" else e.dst_device for e in events]
    for e, d in zip(events, devs):
        if not 0 <= d < num_devices_total:
            raise _device_error(events)(e.seq, d, num_devices_total)
    out = [[] for _ in range(num_devices_total)]
    if not events:
        return out
    keys = np.array(devs, dtype=np.uint32)
    perm = np.zeros(keys.size, dtype=np.uint32)
    L = _lib.lib()
    L.b2l_stable_sort_u32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    _lib.check(L.b2l_stable_sort_u32(keys.ctypes.data, keys.size, perm.ctypes.data), "b2l_stable_sort_u32")
    for i in perm.tolist():
        out[devs[i]].append(events[i])
    return out


# ------------------------------------------------------------------------ DD / RT
def _hashed(data_op_events, strict):
    rows = [(e, TRANSFER) for e in data_op_events]
    cols = _pseudo(rows, _ndev_of(list(data_op_events)))
    return analyze_columns(cols, strict=strict, flags=FLAG_NO_VALIDATE | FLAG_RAW_HASHED | FLAG_SKIP_ALLOC)


def find_duplicate_transfers(data_op_events: Sequence):
    if not data_op_events:
        return []
    T = _family(data_op_events)
    ev = list(data_op_events)
    cf = _hashed(ev, False)
    off, mem = cf.dd_offsets.tolist(), cf.dd_members.tolist()
    out = []
    for g in range(len(off) - 1):
        m = [ev[i] for i in mem[off[g]:off[g + 1]]]
        out.append(T.DuplicateGroup(hash=m[0].hash, dest_device=m[0].dst_device, events=m))
    return out


def find_round_trips(data_op_events: Sequence, strict_pseudocode: bool = False):
    if not data_op_events:
        return []
    T = _family(data_op_events)
    ev = list(data_op_events)
    cf = _hashed(ev, strict_pseudocode)
    off, tx, rx = cf.rt_offsets.tolist(), cf.rt_tx.tolist(), cf.rt_rx.tolist()
    out = []
    for g in range(len(off) - 1):
        trips = [(ev[tx[t]], ev[rx[t]]) for t in range(off[g], off[g + 1])]
        t0 = trips[0][0]
        out.append(T.RoundTripGroup(hash=t0.hash, src_device=t0.src_device, dest_device=t0.dst_device, trips=trips))
    return out


# ------------------------------------------------------------------------ RA / UA / UT
def find_repeated_allocs(data_op_events: Sequence, warn: Optional[Callable] = None):
    if not data_op_events:
        return []
    T = _family(data_op_events)
    cf, ev, pairs = _pairs_from(list(data_op_events), T, warn)
    off, rp = cf.ra_offsets.tolist(), cf.ra_pairs.tolist()
    out = []
    for g in range(len(off) - 1):
        ps = [pairs[r] for r in rp[off[g]:off[g + 1]]]
        a0 = ps[0].alloc_event
        out.append(T.RepeatedAllocGroup(host_addr=a0.src_addr, tgt_device=a0.dst_device, bytes=a0.bytes, pairs=ps))
    return out


def _check_devices(events, ndev, T=None):
    for e in events:
        if not 0 <= e.dst_device < ndev:
            raise _device_error(events)(e.seq, e.dst_device, ndev)


def find_unused_allocs(tgt_events: Sequence, data_op_events: Sequence, num_devices_total: int,
                       warn: Optional[Callable] = None):
    T = _family(list(data_op_events) or list(tgt_events))
    _check_devices(list(tgt_events), num_devices_total, T)
    if not data_op_events:
        return []
    kernels = [(e, KERNEL) for e in tgt_events]
    # every pair's device must be a valid device slot for the per-device sweep (prep.sort_by_device)
    allocs = [e for e in data_op_events if _kind(e) == ALLOC]
    _check_devices(allocs, num_devices_total, T)
    cf, ev, pairs = _pairs_from(list(data_op_events), T, warn, extra_rows=kernels, ndev=num_devices_total,
                                flags=FLAG_SKIP_DDRT)
    return [pairs[r] for r in cf.ua_pairs.tolist()]


def find_unused_transfers(tgt_events: Sequence, data_op_events: Sequence, num_devices_total: int):
    T = _family(list(data_op_events) or list(tgt_events))
    _check_devices(list(tgt_events), num_devices_total, T)
    _check_devices(list(data_op_events), num_devices_total, T)
    if not data_op_events:
        return []
    rows = [(e, KERNEL) for e in tgt_events] + [(e, TRANSFER) for e in data_op_events]
    order = np.argsort(np.fromiter((e.start_ns for e, _ in rows), dtype=np.uint64, count=len(rows)), kind="stable")
    rows = [rows[i] for i in order]
    cols = _pseudo(rows, num_devices_total)
    cf = analyze_columns(cols, flags=FLAG_NO_VALIDATE | FLAG_SKIP_DDRT)
    return [rows[i][0] for i in cf.ut_events.tolist()]
