"""Drop-in analyzer API backed by the B200 engine (libb2l.so).

Same signatures, results, ordering and errors as the reference:
  analyze(trace, warn=None, strict_pseudocode=False) -> Findings   detectors.py:274-326
  estimate(trace, findings) -> SavingsEstimate                     estimator.py:61-151
  attribute(trace, findings) -> list[AttributedIssue]              report.py:73-95
plus columnar entry points that skip Python objects entirely:
  analyze_columns(cols, strict=False) -> ColumnarFindings
  analyze_many(traces) -> iterator of (ColumnarFindings, ColumnarSavings), uploads overlapped
  savings_columns(cols, cf) -> ColumnarSavings

All detection and all integer sums run in CUDA (b2l_analyze / b2l_savings_compute);
this module only converts between Python objects and columns and builds the
result objects (which reference the caller's own TraceEvent objects, as the
reference does).  The only float arithmetic -- the speedup and pct_of_wall
divisions -- is done here from exact integers, as in the reference.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .columns import Columns, Unrepresentable, loc_key, to_columns
from .errors import FindingsTraceMismatch as _OwnMismatch
from .errors import InvalidTrace as _OwnInvalid
from .types import type_family

CATEGORIES = ("DD", "RT", "RA", "UA", "UT")
INFINITE_SPEEDUP = float("inf")
SYNTHETIC = 0xFFFFFFFF
U64_MAX = 2**64 - 1
WARN_REASON = "delete without a live allocation at this device address"  # prep.py:75-76

# ------------------------------------------------------------------------ C structs (include/b2l.h)
_P = ctypes.c_void_p
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_i32 = ctypes.c_int32


class _Cols(ctypes.Structure):
    _fields_ = [("n_events", _u64), ("num_devices_total", _i32), ("host_device", _i32),
                ("seq", _P), ("start_ns", _P), ("end_ns", _P), ("src_addr", _P), ("dst_addr", _P),
                ("bytes", _P), ("hash", _P), ("src_device", _P), ("dst_device", _P), ("kind", _P),
                ("loc", _P), ("n_locs", _u32), ("loc_flags", _P), ("loc_bucket", _P), ("n_buckets", _u32),
                ("device_resident", _i32)]


class _Findings(ctypes.Structure):
    _fields_ = [("n_events", _u64), ("n_bad", _u64), ("bad_index", _P), ("bad_rules", _P),
                ("dd_groups", _u64), ("dd_offsets", _P), ("dd_members", _P),
                ("rt_groups", _u64), ("rt_offsets", _P), ("rt_tx", _P), ("rt_rx", _P),
                ("n_pairs", _u64), ("pair_alloc", _P), ("pair_delete", _P), ("synthetic_end_ns", _u64),
                ("n_warnings", _u64), ("warn_index", _P),
                ("ra_groups", _u64), ("ra_offsets", _P), ("ra_pairs", _P),
                ("n_ua", _u64), ("ua_pairs", _P), ("n_ut", _u64), ("ut_events", _P), ("internal", _P)]


class _U128(ctypes.Structure):
    _fields_ = [("lo", _u64), ("hi", _u64)]


class _Savings(ctypes.Structure):
    _fields_ = [("per_category_ns", _U128 * 5), ("union_ns", _U128), ("n_union", _u64), ("union_index", _P),
                ("has_overlaps", _i32), ("min_start_ns", _u64), ("max_end_ns", _u64), ("n_buckets", _u32),
                ("attr_count", _P), ("attr_ns", _P), ("attr_bytes", _P), ("attr_first", _P), ("internal", _P)]


_declared = False


def _L():
    global _declared
    L = _lib.lib()
    if not _declared:
        L.b2l_analyze.argtypes = [ctypes.POINTER(_Cols), _u32, ctypes.POINTER(ctypes.POINTER(_Findings))]
        L.b2l_analyze.restype = ctypes.c_int
        L.b2l_analyze_ex.argtypes = [ctypes.POINTER(_Cols), _u32, _u64, ctypes.POINTER(ctypes.POINTER(_Findings))]
        L.b2l_analyze_ex.restype = ctypes.c_int
        L.b2l_findings_free.argtypes = [ctypes.POINTER(_Findings)]
        L.b2l_findings_free.restype = None
        L.b2l_savings_compute.argtypes = [ctypes.POINTER(_Cols), ctypes.POINTER(_Findings),
                                          ctypes.POINTER(ctypes.POINTER(_Savings))]
        L.b2l_savings_compute.restype = ctypes.c_int
        L.b2l_savings_free.argtypes = [ctypes.POINTER(_Savings)]
        L.b2l_savings_free.restype = None
        L.b2l_lookup_seqs.argtypes = [ctypes.POINTER(_Cols), _P, _u64, _P]
        L.b2l_lookup_seqs.restype = ctypes.c_int
        _declared = True
    return L


def _cols_struct(c: Columns):
    keep = [c.seq, c.start_ns, c.end_ns, c.src_addr, c.dst_addr, c.bytes, c.hash, c.src_device, c.dst_device,
            c.kind, c.loc, c.loc_flags, c.loc_bucket]
    ptr = lambda a: a.ctypes.data if a.size else None  # noqa: E731
    s = _Cols(n_events=c.n, num_devices_total=c.num_devices_total, host_device=c.host_device,
              seq=ptr(c.seq), start_ns=ptr(c.start_ns), end_ns=ptr(c.end_ns), src_addr=ptr(c.src_addr),
              dst_addr=ptr(c.dst_addr), bytes=ptr(c.bytes), hash=ptr(c.hash), src_device=ptr(c.src_device),
              dst_device=ptr(c.dst_device), kind=ptr(c.kind), loc=ptr(c.loc), n_locs=int(c.loc_flags.size),
              loc_flags=ptr(c.loc_flags), loc_bucket=ptr(c.loc_bucket), n_buckets=c.n_buckets,
              device_resident=0)
    return s, keep


def pinned_columns(cols: Columns) -> Columns:
    """A copy of host columns in page-locked memory, so the engine's host->device upload runs
    at full DMA rate (the caller keeps host buffers; the engine still copies them per call)."""
    import dataclasses

    import torch
    rep = {}
    for f in DeviceColumns.FIELDS:
        a = np.ascontiguousarray(getattr(cols, f))
        buf = torch.empty(max(a.nbytes, 1), dtype=torch.uint8, pin_memory=True)
        v = buf.numpy()[:a.nbytes].view(a.dtype)
        v[...] = a
        rep[f] = v
    return dataclasses.replace(cols, **rep)


class DeviceColumns:
    """Columns resident in device memory (torch tensors used only as buffers);
    b2l_analyze reads them in place (device_resident = 1)."""

    FIELDS = ("seq", "start_ns", "end_ns", "src_addr", "dst_addr", "bytes", "hash", "src_device", "dst_device",
              "kind", "loc", "loc_flags", "loc_bucket")

    def __init__(self, cols: Columns, device="cuda", stream=None):
        """Upload host columns; with ``stream`` the copies are queued on it (asynchronous from
        page-locked memory) and ``ready`` is an event recorded after them."""
        import contextlib

        import torch
        self.host = cols
        self.t = {}
        self.ready = None
        ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
        with ctx:
            for f in self.FIELDS:
                a = getattr(cols, f)
                if a.dtype == np.uint64:
                    a = a.view(np.int64)
                elif a.dtype == np.uint32:
                    a = a.view(np.int32)
                self.t[f] = torch.from_numpy(np.ascontiguousarray(a)).to(device, non_blocking=stream is not None)
            if stream is not None:
                self.ready = torch.cuda.Event()
                self.ready.record(stream)
        ptr = lambda f: self.t[f].data_ptr() if self.t[f].numel() else None  # noqa: E731
        self.struct = _Cols(n_events=cols.n, num_devices_total=cols.num_devices_total, host_device=cols.host_device,
                            seq=ptr("seq"), start_ns=ptr("start_ns"), end_ns=ptr("end_ns"), src_addr=ptr("src_addr"),
                            dst_addr=ptr("dst_addr"), bytes=ptr("bytes"), hash=ptr("hash"),
                            src_device=ptr("src_device"), dst_device=ptr("dst_device"), kind=ptr("kind"),
                            loc=ptr("loc"), n_locs=int(cols.loc_flags.size), loc_flags=ptr("loc_flags"),
                            loc_bucket=ptr("loc_bucket"), n_buckets=cols.n_buckets, device_resident=1)

    @property
    def n(self):
        return self.host.n

    @classmethod
    def from_device(cls, t: dict, n: int, like: "DeviceColumns"):
        """Columns already on the device (``t``: field -> tensor, u64 fields as int64, u32 as
        int32), with the location table and trace metadata of ``like``."""
        import dataclasses
        self = cls.__new__(cls)
        meta = like.host
        self.host = dataclasses.replace(meta, n=n)  # metadata only: field arrays belong to `like`
        self.t = dict(t)
        self.t["loc_flags"], self.t["loc_bucket"] = like.t["loc_flags"], like.t["loc_bucket"]
        ptr = lambda f: self.t[f].data_ptr() if self.t[f].numel() and n else None  # noqa: E731
        self.struct = _Cols(n_events=n, num_devices_total=meta.num_devices_total, host_device=meta.host_device,
                            seq=ptr("seq"), start_ns=ptr("start_ns"), end_ns=ptr("end_ns"), src_addr=ptr("src_addr"),
                            dst_addr=ptr("dst_addr"), bytes=ptr("bytes"), hash=ptr("hash"),
                            src_device=ptr("src_device"), dst_device=ptr("dst_device"), kind=ptr("kind"),
                            loc=ptr("loc"), n_locs=int(meta.loc_flags.size),
                            loc_flags=like.t["loc_flags"].data_ptr() if like.t["loc_flags"].numel() else None,
                            loc_bucket=like.t["loc_bucket"].data_ptr() if like.t["loc_bucket"].numel() else None,
                            n_buckets=meta.n_buckets, device_resident=1)
        return self


_COPY_STREAMS: dict = {}


def analyze_many(traces, strict: bool = False, device=None, with_savings: bool = True):
    """Analyse a sequence of host traces (Columns), yielding ``(ColumnarFindings,
    ColumnarSavings | None)`` per trace, in order.  Trace k+1's columns are queued for upload on
    a copy stream before trace k is analysed, so from page-locked host memory (``pinned_columns``)
    the host->device traffic hides behind the analysis: the per-trace cost becomes
    max(upload, analysis) instead of their sum.  Every trace's columns are still copied to the
    device and its results back to the host (pageable columns upload synchronously: correct,
    just not overlapped)."""
    import torch
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    # one copy stream per device for every call: the uploads' blocks come from the caching
    # allocator's pool of that stream, so a later call reuses them instead of allocating afresh
    if os.environ.get("B2L_MANY_FRESH_STREAM"):
        copy = torch.cuda.Stream(dev)
    else:
        copy = _COPY_STREAMS.get(dev.index)
        if copy is None:
            copy = _COPY_STREAMS[dev.index] = torch.cuda.Stream(dev)
    it = iter(traces)
    nxt = None
    for cols in it:
        nxt = DeviceColumns(cols, dev, stream=copy)
        break
    while nxt is not None:
        cur, nxt = nxt, None
        for cols in it:  # queue the next upload before this trace's analysis
            nxt = DeviceColumns(cols, dev, stream=copy)
            break
        cur.ready.synchronize()  # this trace's columns are on the device
        cf = analyze_columns(cur, strict=strict, with_savings=with_savings)
        sv = savings_columns(cur, cf) if with_savings else None
        del cur  # analysed (the engine call is synchronous): its buffers may be reused
        yield cf, sv


def _view(ptr, n, dtype, owner):
    """Zero-copy numpy view of engine-owned (pinned) memory; the view keeps `owner` alive."""
    if not n or not ptr:
        return np.zeros(0, dtype=dtype)
    buf = (ctypes.c_char * (int(n) * np.dtype(dtype).itemsize)).from_address(ptr)
    buf._owner = owner
    return np.frombuffer(buf, dtype=dtype)


def _arr(ptr, n, dtype):
    if not n or not ptr:
        return np.zeros(0, dtype=dtype)
    size = int(n) * np.dtype(dtype).itemsize
    buf = (ctypes.c_char * size).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype).copy()


# ------------------------------------------------------------------------ columnar results
@dataclass
class ColumnarFindings:
    """Findings as index arrays (see include/b2l.h b2l_findings)."""
    n_events: int
    dd_offsets: np.ndarray
    dd_members: np.ndarray
    rt_offsets: np.ndarray
    rt_tx: np.ndarray
    rt_rx: np.ndarray
    pair_alloc: np.ndarray
    pair_delete: np.ndarray
    synthetic_end_ns: int
    warn_index: np.ndarray
    ra_offsets: np.ndarray
    ra_pairs: np.ndarray
    ua_pairs: np.ndarray
    ut_events: np.ndarray
    _handle: object = None  # engine-side findings (device copies) -- reused by savings

    def counts(self):
        return {"DD": len(self.dd_offsets) - 1, "RT": len(self.rt_offsets) - 1, "RA": len(self.ra_offsets) - 1,
                "UA": len(self.ua_pairs), "UT": len(self.ut_events)}


class _Handle:
    """Owns a b2l_findings* until garbage-collected."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr:
                _L().b2l_findings_free(self.ptr)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass
        self.ptr = None


class EngineInvalid(Exception):
    def __init__(self, bad_index, bad_rules):
        super().__init__("invalid trace")
        self.bad_index = bad_index
        self.bad_rules = bad_rules


FLAG_STRICT_RT, FLAG_VALIDATE_ONLY, FLAG_SYNTH_END, FLAG_SKIP_DDRT, FLAG_SKIP_ALLOC = 1, 2, 4, 8, 16
FLAG_WITH_SAVINGS = 128


def analyze_columns(cols: Columns, strict: bool = False, flags: int = 0,
                    synthetic_end_ns: Optional[int] = None, with_savings: bool = False) -> ColumnarFindings:
    """Run the whole detection pipeline on the device.  Raises EngineInvalid with
    the flagged events / rule bits when the trace fails validation.  ``flags`` /
    ``synthetic_end_ns`` are the shard controls of b2l_analyze_ex (sharded.py).
    ``with_savings``: the same call also computes the estimate/attribute aggregates, feeding
    each category in as its detector chain finishes; the next ``savings_columns`` of the same
    columns returns them without another pass."""
    if with_savings:
        flags |= FLAG_WITH_SAVINGS
    L = _L()
    if isinstance(cols, DeviceColumns):
        cs, keep = cols.struct, None
    else:
        cs, keep = _cols_struct(cols)
    fp = ctypes.POINTER(_Findings)()
    fl = flags | (FLAG_STRICT_RT if strict else 0)
    if synthetic_end_ns is not None:
        fl |= FLAG_SYNTH_END
    rc = L.b2l_analyze_ex(ctypes.byref(cs), fl, int(synthetic_end_ns or 0), ctypes.byref(fp))
    handle = _Handle(fp if fp else None)
    del keep
    if rc == _lib.B2L_E_INVALID_TRACE:
        f = fp.contents
        raise EngineInvalid(_arr(f.bad_index, f.n_bad, np.uint32), _arr(f.bad_rules, f.n_bad, np.uint32))
    _lib.check(rc, "b2l_analyze")
    f = fp.contents
    if flags & FLAG_VALIDATE_ONLY:
        return None
    V = lambda ptr, n, dt: _view(ptr, n, dt, handle)  # noqa: E731
    dd_off = V(f.dd_offsets, f.dd_groups + 1, np.uint64)
    rt_off = V(f.rt_offsets, f.rt_groups + 1, np.uint64)
    ra_off = V(f.ra_offsets, f.ra_groups + 1, np.uint64)
    nm, nt, nr = (int(o[-1]) if len(o) else 0 for o in (dd_off, rt_off, ra_off))
    return ColumnarFindings(
        n_events=f.n_events, dd_offsets=dd_off, dd_members=V(f.dd_members, nm, np.uint32),
        rt_offsets=rt_off, rt_tx=V(f.rt_tx, nt, np.uint32), rt_rx=V(f.rt_rx, nt, np.uint32),
        pair_alloc=V(f.pair_alloc, f.n_pairs, np.uint32), pair_delete=V(f.pair_delete, f.n_pairs, np.uint32),
        synthetic_end_ns=int(f.synthetic_end_ns), warn_index=V(f.warn_index, f.n_warnings, np.uint32),
        ra_offsets=ra_off, ra_pairs=V(f.ra_pairs, nr, np.uint32),
        ua_pairs=V(f.ua_pairs, f.n_ua, np.uint32), ut_events=V(f.ut_events, f.n_ut, np.uint32),
        _handle=handle)


@dataclass
class ColumnarSavings:
    per_category_ns: dict
    union_ns: int
    union_index: np.ndarray
    has_overlaps: bool
    min_start_ns: int
    max_end_ns: int
    attr_count: np.ndarray   # [5, n_buckets]
    attr_ns: list            # [5][n_buckets] python ints
    attr_bytes: list
    attr_first: np.ndarray   # [5, n_buckets] (pos << 32 | event), UINT64_MAX = empty


def _u128(v) -> int:
    return int(v.lo) | (int(v.hi) << 64)


def _findings_struct(cf: ColumnarFindings):
    keep = []

    def p(a):
        a = np.ascontiguousarray(a)
        keep.append(a)
        return a.ctypes.data if a.size else None
    s = _Findings(n_events=cf.n_events, n_bad=0, bad_index=None, bad_rules=None,
                  dd_groups=len(cf.dd_offsets) - 1, dd_offsets=p(cf.dd_offsets.astype(np.uint64)),
                  dd_members=p(cf.dd_members.astype(np.uint32)),
                  rt_groups=len(cf.rt_offsets) - 1, rt_offsets=p(cf.rt_offsets.astype(np.uint64)),
                  rt_tx=p(cf.rt_tx.astype(np.uint32)), rt_rx=p(cf.rt_rx.astype(np.uint32)),
                  n_pairs=len(cf.pair_alloc), pair_alloc=p(cf.pair_alloc.astype(np.uint32)),
                  pair_delete=p(cf.pair_delete.astype(np.uint32)), synthetic_end_ns=cf.synthetic_end_ns,
                  n_warnings=0, warn_index=None,
                  ra_groups=len(cf.ra_offsets) - 1, ra_offsets=p(cf.ra_offsets.astype(np.uint64)),
                  ra_pairs=p(cf.ra_pairs.astype(np.uint32)),
                  n_ua=len(cf.ua_pairs), ua_pairs=p(cf.ua_pairs.astype(np.uint32)),
                  n_ut=len(cf.ut_events), ut_events=p(cf.ut_events.astype(np.uint32)), internal=None)
    return s, keep


def savings_columns(cols: Columns, cf: ColumnarFindings) -> ColumnarSavings:
    """Exact integer estimate/attribute aggregates on the device."""
    L = _L()
    if isinstance(cols, DeviceColumns):
        cs, keep_c = cols.struct, None
    else:
        cs, keep_c = _cols_struct(cols)
    if cf._handle is not None and cf._handle.ptr:
        fptr = cf._handle.ptr
        keep_f = None
    else:
        fs, keep_f = _findings_struct(cf)
        fptr = ctypes.pointer(fs)
    sp = ctypes.POINTER(_Savings)()
    rc = L.b2l_savings_compute(ctypes.byref(cs), fptr, ctypes.byref(sp))
    owner = _SavingsHandle(sp if sp else None)
    _lib.check(rc, "b2l_savings_compute")
    s = sp.contents
    nb = int(s.n_buckets)
    per = {c: _u128(s.per_category_ns[k]) for k, c in enumerate(CATEGORIES)}
    ns = _arr(s.attr_ns, 2 * 5 * nb, np.uint64).reshape(5, nb, 2) if nb else np.zeros((5, 0, 2), np.uint64)
    by = _arr(s.attr_bytes, 2 * 5 * nb, np.uint64).reshape(5, nb, 2) if nb else np.zeros((5, 0, 2), np.uint64)
    out = ColumnarSavings(
        per_category_ns=per, union_ns=_u128(s.union_ns),
        union_index=_view(s.union_index, s.n_union, np.uint32, owner),  # zero-copy (pinned)
        has_overlaps=bool(s.has_overlaps), min_start_ns=int(s.min_start_ns), max_end_ns=int(s.max_end_ns),
        attr_count=_arr(s.attr_count, 5 * nb, np.uint64).reshape(5, nb),
        attr_ns=[[int(ns[c, b, 0]) | (int(ns[c, b, 1]) << 64) for b in range(nb)] for c in range(5)],
        attr_bytes=[[int(by[c, b, 0]) | (int(by[c, b, 1]) << 64) for b in range(nb)] for c in range(5)],
        attr_first=_arr(s.attr_first, 5 * nb, np.uint64).reshape(5, nb))
    del keep_c, keep_f
    return out


class _SavingsHandle:
    """Owns a b2l_savings* (its pinned arrays back zero-copy views) until garbage-collected."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr:
                _L().b2l_savings_free(self.ptr)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass
        self.ptr = None


def lookup_seqs(cols: Columns, seqs: np.ndarray) -> np.ndarray:
    L = _L()
    cs, keep = _cols_struct(cols)
    q = np.ascontiguousarray(seqs, dtype=np.uint64)
    out = np.zeros(q.size, dtype=np.uint32)
    rc = L.b2l_lookup_seqs(ctypes.byref(cs), q.ctypes.data if q.size else None, q.size,
                           out.ctypes.data if q.size else None)
    _lib.check(rc, "b2l_lookup_seqs")
    del keep
    return out


# ------------------------------------------------------------------------ violations (model.py:125-200)
_RULE_TEXT = [
    (1 << 0, "interval", lambda e, nd: f"start_ns {e.start_ns} > end_ns {e.end_ns}"),
    (1 << 1, "device", lambda e, nd: f"src_device={e.src_device} out of range [0,{nd})"),
    (1 << 2, "device", lambda e, nd: f"dst_device={e.dst_device} out of range [0,{nd})"),
    (1 << 3, "transfer", lambda e, nd: "non-empty transfer has no content hash"),
    (1 << 4, "alloc", lambda e, nd: "allocation of zero bytes"),
    (1 << 5, "alloc", lambda e, nd: "allocation with null device address"),
    (1 << 6, "delete", lambda e, nd: "deletion with null device address"),
    (1 << 7, "kernel", lambda e, nd: "kernel src_device must equal dst_device"),
    (1 << 8, "location", lambda e, nd: "file present but line missing"),
    (1 << 9, "location", lambda e, nd: f"line={e.loc.line} must be positive"),
    (1 << 10, "order", lambda e, nd: "events not sorted by (start_ns, seq)"),
    (1 << 11, "order", lambda e, nd: "seq values not strictly increasing"),
]


def _header_violations(trace, V):
    out = []
    nd = trace.num_devices_total
    if nd < 1:
        out.append(V("header", f"num_devices_total={nd} must be positive"))
    if not 0 <= trace.host_device < max(nd, 1):
        out.append(V("header", f"host_device={trace.host_device} out of range"))
    w = trace.wall_time_ns
    if w is not None and (not isinstance(w, int) or isinstance(w, bool) or not 0 <= w <= U64_MAX):
        out.append(V("field-range", f"wall_time_ns={w!r} is not a 64-bit unsigned value", None))
    return out


def _event_violations(trace, bad_index, bad_rules, V):
    out = []
    nd = trace.num_devices_total
    for i, m in zip(bad_index.tolist(), bad_rules.tolist()):
        e = trace.events[i]
        for bit, rule, text in _RULE_TEXT:
            if m & bit:
                out.append(V(rule, text(e, nd), e.seq))
    return out


def _boundary_violations(trace, V):
    """Traces whose values cannot be carried by the u64/i32 device columns (negative,
    >= 2**64, non-int fields).  Such a trace is invalid by construction; the
    violation list is produced at the boundary, in model.py:125-200's order."""
    out = _header_violations(trace, V)
    nd = trace.num_devices_total
    prev_start, prev_seq = -1, -1

    def bad64(x):
        return not isinstance(x, int) or isinstance(x, bool) or not 0 <= x <= U64_MAX
    for e in trace.events:
        seq = e.seq
        for name in ("seq", "start_ns", "end_ns", "src_addr", "dst_addr", "bytes", "hash"):
            x = getattr(e, name)
            if bad64(x):
                out.append(V("field-range", f"{name}={x!r} is not a 64-bit unsigned value", seq))
        if e.start_ns > e.end_ns:
            out.append(V("interval", f"start_ns {e.start_ns} > end_ns {e.end_ns}", seq))
        if not 0 <= e.src_device < nd:
            out.append(V("device", f"src_device={e.src_device} out of range [0,{nd})", seq))
        if not 0 <= e.dst_device < nd:
            out.append(V("device", f"dst_device={e.dst_device} out of range [0,{nd})", seq))
        k = getattr(e.kind, "value", e.kind)
        if k == "transfer":
            if e.bytes > 0 and e.hash == 0:
                out.append(V("transfer", "non-empty transfer has no content hash", seq))
        elif k == "alloc":
            if e.bytes <= 0:
                out.append(V("alloc", "allocation of zero bytes", seq))
            if e.dst_addr == 0:
                out.append(V("alloc", "allocation with null device address", seq))
        elif k == "delete":
            if e.dst_addr == 0:
                out.append(V("delete", "deletion with null device address", seq))
        elif k == "kernel":
            if e.src_device != e.dst_device:
                out.append(V("kernel", "kernel src_device must equal dst_device", seq))
        if e.loc.file is not None and e.loc.line is None:
            out.append(V("location", "file present but line missing", seq))
        if e.loc.line is not None and e.loc.line <= 0:
            out.append(V("location", f"line={e.loc.line} must be positive", seq))
        if e.start_ns < prev_start or (e.start_ns == prev_start and seq < prev_seq):
            out.append(V("order", "events not sorted by (start_ns, seq)", seq))
        if seq <= prev_seq:
            out.append(V("order", "seq values not strictly increasing", seq))
        prev_start, prev_seq = e.start_ns, seq
    return out


# ------------------------------------------------------------------------ drop-in API
_RECENT: dict = {}  # id(Findings) -> (findings, trace, cols, ColumnarFindings, shape)  (small LRU)
_RECENT_MAX = 4


def _shape(f):
    return (id(f.duplicates), len(f.duplicates), id(f.round_trips), len(f.round_trips), id(f.repeated_allocs),
            len(f.repeated_allocs), id(f.unused_allocs), len(f.unused_allocs), id(f.unused_transfers),
            len(f.unused_transfers))


def _remember(f, trace, cols, cf):
    _RECENT[id(f)] = (f, trace, cols, cf, _shape(f))
    while len(_RECENT) > _RECENT_MAX:
        _RECENT.pop(next(iter(_RECENT)))


def analyze(trace, warn: Optional[Callable] = None, strict_pseudocode: bool = False):
    """dmlens.detectors.analyze drop-in (detectors.py:274-326)."""
    T = type_family(trace)
    Invalid = T.InvalidTrace or _OwnInvalid
    try:
        cols = to_columns(trace)
    except Unrepresentable:
        raise Invalid(_boundary_violations(trace, T.Violation))
    head = _header_violations(trace, T.Violation)
    try:
        cf = analyze_columns(cols, strict=strict_pseudocode, with_savings=True)
    except EngineInvalid as exc:
        raise Invalid(head + _event_violations(trace, exc.bad_index, exc.bad_rules, T.Violation))
    if head:
        raise Invalid(head)
    findings = _materialize(trace, cols, cf, T, warn)
    _remember(findings, trace, cols, cf)
    return findings


def _materialize(trace, cols, cf: ColumnarFindings, T, warn):
    ev = trace.events
    if warn is not None:
        for i in cf.warn_index.tolist():
            warn(T.PrepWarning(ev[i].seq, WARN_REASON))
    pairs = []
    delete_kind = T.EventKind.DELETE
    end = cf.synthetic_end_ns
    for a, d in zip(cf.pair_alloc.tolist(), cf.pair_delete.tolist()):
        al = ev[a]
        if d == SYNTHETIC:
            syn = T.TraceEvent(seq=al.seq, kind=delete_kind, start_ns=end, end_ns=end, src_device=al.src_device,
                               dst_device=al.dst_device, src_addr=0, dst_addr=al.dst_addr, bytes=0, hash=0,
                               loc=al.loc)
            pairs.append(T.AllocPair(al, syn, synthetic_delete=True))
        else:
            pairs.append(T.AllocPair(al, ev[d]))
    dd = []
    off = cf.dd_offsets.tolist()
    mem = cf.dd_members.tolist()
    for g in range(len(off) - 1):
        members = [ev[i] for i in mem[off[g]:off[g + 1]]]
        dd.append(T.DuplicateGroup(hash=members[0].hash, dest_device=members[0].dst_device, events=members))
    rt = []
    off = cf.rt_offsets.tolist()
    tx, rx = cf.rt_tx.tolist(), cf.rt_rx.tolist()
    for g in range(len(off) - 1):
        trips = [(ev[tx[t]], ev[rx[t]]) for t in range(off[g], off[g + 1])]
        t0 = trips[0][0]
        rt.append(T.RoundTripGroup(hash=t0.hash, src_device=t0.src_device, dest_device=t0.dst_device, trips=trips))
    ra = []
    off = cf.ra_offsets.tolist()
    rp = cf.ra_pairs.tolist()
    for g in range(len(off) - 1):
        ps = [pairs[r] for r in rp[off[g]:off[g + 1]]]
        a0 = ps[0].alloc_event
        ra.append(T.RepeatedAllocGroup(host_addr=a0.src_addr, tgt_device=a0.dst_device, bytes=a0.bytes, pairs=ps))
    ua = [pairs[r] for r in cf.ua_pairs.tolist()]
    ut = [ev[i] for i in cf.ut_events.tolist()]
    return T.Findings(duplicates=dd, round_trips=rt, repeated_allocs=ra, unused_allocs=ua, unused_transfers=ut)


def _columnar_from_objects(trace, cols, findings, T):
    """Findings objects -> index arrays, by seq lookup on the device (estimator.py:72-75:
    findings may only reference seqs present in the trace)."""
    Mismatch = T.FindingsTraceMismatch or _OwnMismatch
    seqs = []
    for g in findings.duplicates:
        seqs.extend(e.seq for e in g.events)
    for g in findings.round_trips:
        for a, b in g.trips:
            seqs.append(a.seq)
            seqs.append(b.seq)

    def pair_seqs(p):
        seqs.append(p.alloc_event.seq)
        if not p.synthetic_delete:
            seqs.append(p.delete_event.seq)
    for g in findings.repeated_allocs:
        for p in g.pairs:
            pair_seqs(p)
    for p in findings.unused_allocs:
        pair_seqs(p)
    seqs.extend(e.seq for e in findings.unused_transfers)
    bad = [s for s in seqs if not isinstance(s, int) or not 0 <= s <= U64_MAX]
    if bad:
        raise Mismatch(bad[0])
    idx = lookup_seqs(cols, np.array(seqs, dtype=np.uint64)) if seqs else np.zeros(0, np.uint32)
    missing = np.nonzero(idx == SYNTHETIC)[0]
    if missing.size:
        raise Mismatch(seqs[int(missing[0])])
    it = iter(idx.tolist())
    dd_off, dd_mem = [0], []
    for g in findings.duplicates:
        dd_mem.extend(next(it) for _ in g.events)
        dd_off.append(len(dd_mem))
    rt_off, rt_tx, rt_rx = [0], [], []
    for g in findings.round_trips:
        for _ in g.trips:
            rt_tx.append(next(it))
            rt_rx.append(next(it))
        rt_off.append(len(rt_tx))
    pa, pd = [], []

    def pair_index(p):
        pa.append(next(it))
        pd.append(SYNTHETIC if p.synthetic_delete else next(it))
        return len(pa) - 1
    ra_off, ra_pairs = [0], []
    for g in findings.repeated_allocs:
        ra_pairs.extend(pair_index(p) for p in g.pairs)
        ra_off.append(len(ra_pairs))
    ua = [pair_index(p) for p in findings.unused_allocs]
    ut = [next(it) for _ in findings.unused_transfers]
    u32 = lambda x: np.array(x, dtype=np.uint32)  # noqa: E731
    u64 = lambda x: np.array(x, dtype=np.uint64)  # noqa: E731
    return ColumnarFindings(n_events=cols.n, dd_offsets=u64(dd_off), dd_members=u32(dd_mem), rt_offsets=u64(rt_off),
                            rt_tx=u32(rt_tx), rt_rx=u32(rt_rx), pair_alloc=u32(pa), pair_delete=u32(pd),
                            synthetic_end_ns=0, warn_index=u32([]), ra_offsets=u64(ra_off), ra_pairs=u32(ra_pairs),
                            ua_pairs=u32(ua), ut_events=u32(ut))


def _savings_for(trace, findings):
    T = type_family(trace)
    hit = _RECENT.get(id(findings))
    if hit is not None and hit[0] is findings and hit[1] is trace and hit[4] == _shape(findings):
        _, _, cols, cf, _ = hit
    else:
        cols = to_columns(trace)
        cf = _columnar_from_objects(trace, cols, findings, T)
    return T, cols, savings_columns(cols, cf)


def _wall(trace, sv: ColumnarSavings):
    if trace.wall_time_ns is not None:
        return trace.wall_time_ns
    if not trace.events:
        return 0
    return sv.max_end_ns - sv.min_start_ns


def estimate(trace, findings):
    """dmlens.estimator.estimate drop-in (estimator.py:61-151)."""
    T, cols, sv = _savings_for(trace, findings)
    warnings = []
    union_ns = sv.union_ns
    wall = _wall(trace, sv)
    if union_ns > wall:
        warnings.append(f"eliminable time {union_ns} ns exceeds wall time {wall} ns; clamped to wall time")
        union_ns = wall
    if union_ns < 0:
        warnings.append("negative eliminable time clamped to 0")
        union_ns = 0
    if union_ns == 0:
        speedup = 1.0
    elif union_ns == wall:
        warnings.append("eliminable time equals wall time; predicted speedup is unbounded")
        speedup = INFINITE_SPEEDUP
    else:
        speedup = wall / (wall - union_ns)
    if sv.has_overlaps:
        warnings.append("trace contains overlapping event intervals; savings assume serialized "
                        "operations and may be unreliable")
    ev = trace.events
    return T.SavingsEstimate(per_category_ns=dict(sv.per_category_ns), union_ns=union_ns, wall_time_ns=wall,
                             predicted_speedup=speedup, eliminable_seqs=frozenset(ev[i].seq
                                                                                 for i in sv.union_index.tolist()),
                             warnings=tuple(warnings))


def attribute(trace, findings):
    """dmlens.report.attribute drop-in (report.py:73-95)."""
    T, cols, sv = _savings_for(trace, findings)
    wall = _wall(trace, sv)
    ev = trace.events
    issues = []
    for c, cat in enumerate(CATEGORIES):
        rows = []
        for b in np.nonzero(sv.attr_count[c])[0].tolist():
            first_ev = int(sv.attr_first[c, b]) & 0xFFFFFFFF
            loc = ev[first_ev].loc
            total_ns = sv.attr_ns[c][b]
            rows.append(T.AttributedIssue(category=cat, location=loc, occurrence_count=int(sv.attr_count[c, b]),
                                          total_ns=total_ns, total_bytes=sv.attr_bytes[c][b],
                                          pct_of_wall=(total_ns / wall) if wall else 0.0))
        rows.sort(key=lambda r: (-r.total_ns, loc_key(r.location.codeptr, r.location.file, r.location.line)))
        issues.extend(rows)
    return issues
