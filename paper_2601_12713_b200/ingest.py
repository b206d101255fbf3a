"""NDJSON trace ingest -- drop-in for dmlens.traceio.parse_trace / load_trace_file
(traceio.py:153-191, 240-242) on the native parser (b2l_ingest_ndjson, C++ over host
threads) plus GPU sorting (b2l_sort_u64_pairs) and GPU validation (b2l_analyze_ex
VALIDATE_ONLY).

  parse_trace(data, types=None) -> Trace            objects, like the reference
  parse_trace_columns(data)     -> Columns          no Python objects (large traces)

Error behaviour is the reference's: MissingHeader, UnsupportedVersion,
MalformedRecord(line_no, reason), InvariantViolation(violations) (classes from
dmlens.traceio when types="dmlens").  The native parser accepts exactly the records
the reference accepts without error and lists the lines it cannot vouch for; only
those lines are checked here the reference's way (``_canonical_line``, restating
traceio.py:153-181 line by line): the first bad one raises the reference's exception
for it, unusual-but-valid ones (Unicode whitespace, ``1.0`` as the version, reordered
or unknown fields, escapes) are rewritten in canonical form, and the patched input is
parsed natively again.  A whole-input Python parse (``_parse_exact``) is left only for
traces the columns cannot represent at all (device ids or line numbers beyond the
i32/i64 columns) -- an error path, since such device ids fail validation.
"""
from __future__ import annotations

import ctypes
import json
import os
from collections import namedtuple
from typing import Optional

import numpy as np

from . import _lib
from .analysis import FLAG_VALIDATE_ONLY, EngineInvalid, _RULE_TEXT, analyze_columns
from .columns import LOC_FILE_NO_LINE, LOC_LINE_NONPOS, Columns, loc_key
from .types import family

U64_MAX = 2**64 - 1
I32_MAX = 2**31 - 1
FORMAT_VERSION = 1
_KINDS = ("transfer", "alloc", "delete", "kernel")
_REQUIRED = ("seq", "kind", "t0", "t1", "src_dev", "dst_dev", "src_addr", "dst_addr", "bytes", "hash", "codeptr")


# ------------------------------------------------------------------------ error classes (traceio.py:42-75)
class TraceIOError(Exception):
    pass


class MalformedRecord(TraceIOError):
    def __init__(self, line_no: int, reason: str):
        super().__init__(f"line {line_no}: {reason}")
        self.line_no = line_no
        self.reason = reason


class MissingHeader(TraceIOError):
    def __init__(self, detail: str = "first non-comment line must be the trace header"):
        super().__init__(detail)


class UnsupportedVersion(TraceIOError):
    def __init__(self, version):
        super().__init__(f"unsupported trace format version {version!r} (supported: {FORMAT_VERSION})")
        self.version = version


class InvalidTrace(TraceIOError):  # traceio.py:72-75: serialize_trace refuses an invalid trace
    def __init__(self, violations):
        super().__init__(f"refusing to serialize invalid trace ({len(violations)} violations)")
        self.violations = violations


class InvariantViolation(TraceIOError):
    def __init__(self, violations):
        lines = "; ".join(str(v) for v in violations[:10])
        more = f" (+{len(violations) - 10} more)" if len(violations) > 10 else ""
        super().__init__(f"trace violates model invariants: {lines}{more}")
        self.violations = violations


def _errors(types):
    if types is not None and getattr(types, "root", None):
        import importlib
        t = importlib.import_module(types.root + ".traceio")
        return t.MalformedRecord, t.MissingHeader, t.UnsupportedVersion, t.InvariantViolation
    return MalformedRecord, MissingHeader, UnsupportedVersion, InvariantViolation


# ------------------------------------------------------------------------ native path
class _Ingest(ctypes.Structure):
    _P = ctypes.c_void_p
    _fields_ = [("err_line", ctypes.c_uint64), ("header_line", ctypes.c_uint64), ("version", ctypes.c_uint64),
                ("num_devices", ctypes.c_uint64), ("host_device", ctypes.c_uint64), ("wall_time_ns", ctypes.c_uint64),
                ("has_wall", ctypes.c_int32), ("n_events", ctypes.c_uint64),
                ("seq", _P), ("start_ns", _P), ("end_ns", _P), ("src_device", _P), ("dst_device", _P),
                ("src_addr", _P), ("dst_addr", _P), ("bytes", _P), ("hash", _P), ("kind", _P), ("loc", _P),
                ("n_locs", ctypes.c_uint32), ("loc_codeptr", _P), ("loc_line", _P), ("loc_file_off", _P),
                ("loc_file_len", _P), ("strings", _P), ("n_err_lines", ctypes.c_uint64), ("err_lines", _P)]


def _as_bytes(data):
    if hasattr(data, "read"):
        data = data.read()
    if isinstance(data, str):
        return data.encode("utf-8"), data
    data = bytes(data)
    return data, None


def _copy(ptr, n, dtype):
    if not n or not ptr:
        return np.zeros(0, dtype=dtype)
    buf = (ctypes.c_char * (int(n) * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype).copy()


class _IngestHandle:
    """Owns a b2l_ingest* until the last column view over its arrays is gone."""

    def __init__(self, L, ptr):
        self.L, self.ptr = L, ptr

    def __del__(self):
        try:
            if self.ptr:
                self.L.b2l_ingest_free(self.ptr)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass
        self.ptr = None


def _view(ptr, n, dtype, owner):
    """Zero-copy numpy view of parser-owned memory that keeps `owner` alive."""
    if not n or not ptr:
        return np.zeros(0, dtype=dtype)
    buf = (ctypes.c_char * (int(n) * np.dtype(dtype).itemsize)).from_address(ptr)
    buf._owner = owner
    return np.frombuffer(buf, dtype=dtype)


_Unvouched = namedtuple("_Unvouched", "header_line lines")


def _native(raw: bytes, threads: int):
    """(header, columns, locs), or _Unvouched(header_line, lines) when the native parser cannot
    vouch for some lines (no columns are returned then)."""
    L = _lib.lib()
    L.b2l_ingest_ndjson.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_int,
                                    ctypes.POINTER(ctypes.POINTER(_Ingest))]
    L.b2l_ingest_ndjson.restype = ctypes.c_int
    L.b2l_ingest_free.argtypes = [ctypes.POINTER(_Ingest)]
    out = ctypes.POINTER(_Ingest)()
    _lib.check(L.b2l_ingest_ndjson(raw, len(raw), threads, ctypes.byref(out)), "b2l_ingest_ndjson")
    handle = _IngestHandle(L, out)  # the event columns below are views over the parser's arrays
    g = out.contents
    if g.err_line:
        return _Unvouched(int(g.header_line), _copy(g.err_lines, int(g.n_err_lines), np.uint64).tolist())
    n = int(g.n_events)
    cols = {f: _view(getattr(g, f), n, np.uint64, handle) for f in
            ("seq", "start_ns", "end_ns", "src_device", "dst_device", "src_addr", "dst_addr", "bytes", "hash")}
    cols["kind"] = _view(g.kind, n, np.uint8, handle)
    cols["loc"] = _view(g.loc, n, np.uint32, handle)
    nl = int(g.n_locs)
    cp = _copy(g.loc_codeptr, nl, np.uint64)
    ln = _copy(g.loc_line, nl, np.int64)
    off = _copy(g.loc_file_off, nl, np.uint64)
    flen = _copy(g.loc_file_len, nl, np.uint32)
    strings = b""
    total = int(max((int(o) + int(fl) for o, fl in zip(off, flen) if o != U64_MAX), default=0))
    if total:
        strings = ctypes.string_at(g.strings, total)
    locs = []
    for k in range(nl):
        f = None if off[k] == U64_MAX else strings[int(off[k]):int(off[k]) + int(flen[k])].decode(
            "utf-8", "surrogatepass")
        locs.append((int(cp[k]), f, None if ln[k] < 0 else int(ln[k])))
    header = (int(g.version), int(g.num_devices), int(g.host_device),
              int(g.wall_time_ns) if g.has_wall else None)
    return header, cols, locs


class _Unrepresentable(Exception):
    """A valid line the columns cannot hold (the canonical rewrite is still not vouched)."""


def _native_checked(raw: bytes, threads: int, types):
    """Native parse; lines it cannot vouch for are checked the reference's way and patched
    (``_canonical_line``) before the next native pass.  Raises the reference's exception for
    the first bad line, or _Unrepresentable."""
    prev = None
    while True:
        got = _native(raw, threads)
        if not isinstance(got, _Unvouched):
            return got
        if got.header_line == 0:
            raise _errors(types)[1]("empty input: no header line found")
        if got == prev:
            raise _Unrepresentable()
        prev = got
        lines = raw.split(b"\n")
        changed = False
        for ln in got.lines:
            new = _canonical_line(lines[ln - 1].decode("utf-8"), ln, ln == got.header_line, types)
            changed |= new != lines[ln - 1]
            lines[ln - 1] = new
        if not changed:
            raise _Unrepresentable()
        raw = b"\n".join(lines)


def _sort_perm(t0: np.ndarray, seq: np.ndarray) -> Optional[np.ndarray]:
    """Permutation sorting events by (t0, seq) (traceio.py:183), or None if already sorted."""
    n = t0.size
    if n < 2:
        return None
    d0 = t0[1:] >= t0[:-1]
    if np.all(d0 & ((t0[1:] > t0[:-1]) | (seq[1:] >= seq[:-1]))):
        return None
    perm = np.zeros(n, dtype=np.uint32)
    L = _lib.lib()
    L.b2l_sort_u64_pairs.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_uint64] + [ctypes.c_void_p]
    L.b2l_sort_u64_pairs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    a, b = np.ascontiguousarray(t0), np.ascontiguousarray(seq)
    _lib.check(L.b2l_sort_u64_pairs(a.ctypes.data, b.ctypes.data, n, perm.ctypes.data), "b2l_sort_u64_pairs")
    return perm


_Ev = namedtuple("_Ev", "seq start_ns end_ns src_device dst_device loc")
_Lc = namedtuple("_Lc", "line")


def _to_columns(header, cols, locs) -> Columns:
    version, nd, host, wall = header
    perm = _sort_perm(cols["start_ns"], cols["seq"])
    if perm is not None:
        cols = {k: v[perm] for k, v in cols.items()}
    n = cols["seq"].size
    if wall is None:  # derived once at parse time (traceio.py:185-186)
        wall = int(cols["end_ns"].max() - cols["start_ns"].min()) if n else 0
    flags, bucket_of, bucket_ids, bucket_keys = [], [], {}, []
    for cp, f, ln in locs:
        fl = (LOC_FILE_NO_LINE if (f is not None and ln is None) else 0) | (
            LOC_LINE_NONPOS if (ln is not None and ln <= 0) else 0)
        flags.append(fl)
        bk = loc_key(cp, f, ln)
        if bk not in bucket_ids:
            bucket_ids[bk] = len(bucket_keys)
            bucket_keys.append(bk)
        bucket_of.append(bucket_ids[bk])
    return Columns(n=n, num_devices_total=nd, host_device=host, seq=cols["seq"], start_ns=cols["start_ns"],
                   end_ns=cols["end_ns"], src_addr=cols["src_addr"], dst_addr=cols["dst_addr"], bytes=cols["bytes"],
                   hash=cols["hash"], src_device=cols["src_device"].astype(np.int32),
                   dst_device=cols["dst_device"].astype(np.int32), kind=cols["kind"], loc=cols["loc"],
                   loc_flags=np.array(flags or [0], dtype=np.uint8), loc_bucket=np.array(bucket_of or [0], np.uint32),
                   n_buckets=max(len(bucket_keys), 1), bucket_keys=bucket_keys or [(1, "", 0)], wall_time_ns=wall,
                   locs=locs or [(0, None, None)])


def _violation_type(types):
    T = family(types.root) if types is not None and getattr(types, "root", None) else family(None)
    return T.Violation


def _header_violations(c: Columns, types):
    V = _violation_type(types)
    out = []
    if c.num_devices_total < 1:
        out.append(V("header", f"num_devices_total={c.num_devices_total} must be positive"))
    if not 0 <= c.host_device < max(c.num_devices_total, 1):
        out.append(V("header", f"host_device={c.host_device} out of range"))
    return out


def event_violations(c: Columns, exc: EngineInvalid, types=None):
    """The reference's Violation list (model.py:133-196 messages, trace order) for the events an
    engine run flagged -- from b2l_analyze's validation, whichever call ran it."""
    V = _violation_type(types)
    out = []
    for i, m in zip(exc.bad_index.tolist(), exc.bad_rules.tolist()):
        loc = c.locs[int(c.loc[i])]
        e = _Ev(int(c.seq[i]), int(c.start_ns[i]), int(c.end_ns[i]), int(c.src_device[i]),
                int(c.dst_device[i]), _Lc(loc[2]))
        for bit, rule, text in _RULE_TEXT:
            if m & bit:
                out.append(V(rule, text(e, c.num_devices_total), e.seq))
    return out


def invariant_error(violations, types=None):
    return _errors(types)[3](violations)


def _validate_columns(c: Columns, types):
    """GPU validation of parsed columns -> violations (model.py:125-200 messages)."""
    out = _header_violations(c, types)
    try:
        analyze_columns(c, flags=FLAG_VALIDATE_ONLY)
    except EngineInvalid as exc:
        out += event_violations(c, exc, types)
    return out


def _representable(got) -> bool:
    (_, nd, host, _), cols, _ = got
    return nd <= I32_MAX and host <= I32_MAX and not (cols["src_device"].size and (
        cols["src_device"].max() > I32_MAX or cols["dst_device"].max() > I32_MAX))


def parse_trace_columns(data, threads: Optional[int] = None, types=None, validate: bool = True) -> Columns:
    """Parse + sort + validate into device-ready columns (no per-event Python objects).
    validate=False leaves the event rules to the caller's next engine run (b2l_analyze validates
    anyway; turn its EngineInvalid into the same error with ``event_violations`` /
    ``invariant_error``) -- header rules are always checked here."""
    raw, text = _as_bytes(data)
    if text is None and not raw.isascii():
        text = raw.decode("utf-8")  # the reference decodes first (UnicodeDecodeError as it does)
    threads = threads or min(32, os.cpu_count() or 1)
    try:
        got = _native_checked(raw, threads, types)
    except _Unrepresentable:
        got = None
    if got is None or not _representable(got):  # error path: see the module docstring
        from .columns import to_columns
        return to_columns(_parse_exact(text if text is not None else raw.decode("utf-8"), types))
    c = _to_columns(*got)
    if not validate and not _header_violations(c, types):
        return c
    viol = _validate_columns(c, types)
    if viol:
        raise _errors(types)[3](viol)
    return c


def parse_trace(data, types=None, threads: Optional[int] = None):
    """Drop-in for dmlens.traceio.parse_trace; ``types=family("dmlens")`` returns dmlens objects."""
    raw, text = _as_bytes(data)
    if text is None:
        text = raw.decode("utf-8")
    T = types or family(None)
    threads = threads or min(32, os.cpu_count() or 1)
    try:
        got = _native_checked(raw, threads, types)
    except _Unrepresentable:
        got = None
    if got is None or not _representable(got):  # error path: see the module docstring
        return _parse_exact(text, types)
    c = _to_columns(*got)
    viol = _validate_columns(c, types)
    if viol:
        raise _errors(types)[3](viol)
    locs = [T.CodeLocation(codeptr=cp, file=f, line=ln) for cp, f, ln in c.locs]
    kinds = [T.EventKind(k) for k in _KINDS]
    L = lambda a: a.tolist()  # noqa: E731
    ev = [T.TraceEvent(q, kinds[k], a, b, s, d, sa, da, nb, h, locs[lo]) for q, k, a, b, s, d, sa, da, nb, h, lo in zip(
        L(c.seq), L(c.kind), L(c.start_ns), L(c.end_ns), L(c.src_device), L(c.dst_device), L(c.src_addr),
        L(c.dst_addr), L(c.bytes), L(c.hash), L(c.loc))]
    return T.Trace(version=got[0][0], num_devices_total=c.num_devices_total, host_device=c.host_device,
                   wall_time_ns=c.wall_time_ns, events=ev)


def load_trace_file(path, types=None):
    with open(path, "rb") as fh:
        return parse_trace(fh.read(), types=types)


# ------------------------------------------------------------------------ serialize (traceio.py:193-245)
def _serialize_errors(types):
    if types is not None and getattr(types, "root", None):
        import importlib
        return importlib.import_module(types.root + ".traceio").InvalidTrace
    return InvalidTrace


def serialize_columns(c: Columns, version=FORMAT_VERSION, threads: Optional[int] = None,
                      validate: bool = True) -> bytes:
    """Canonical NDJSON of columns (b2l_serialize_ndjson over host threads).  Only location
    tails are rendered here (json.dumps, once per location); every event line is written
    natively.  validate=True refuses invalid columns as serialize_trace does (GPU validation)."""
    if validate:
        viol = _validate_columns(c, None)
        if version != FORMAT_VERSION:
            viol.append(_violation_type(None)("header", f"version={version} is not serializable as format "
                                                        f"{FORMAT_VERSION}"))
        if viol:
            raise InvalidTrace(viol)
    header = {"dmlens": version, "num_devices": c.num_devices_total, "host_device": c.host_device}
    if c.wall_time_ns is not None:
        header["wall_time_ns"] = c.wall_time_ns
    head = (json.dumps(header, separators=(",", ":")) + "\n").encode("utf-8")
    locs = c.locs or [(0, None, None)] * max(c.n_locs, 1)
    tails = []
    for cp, f, ln in locs:  # traceio.py:193-210 _event_record's location keys
        rec = {"codeptr": cp}
        if f is not None:
            rec["file"] = f
            rec["line"] = ln
        tails.append(("," + json.dumps(rec, separators=(",", ":"))[1:]).encode("utf-8"))
    off = np.zeros(len(tails) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(t) for t in tails])
    blob = b"".join(tails)
    from .analysis import _cols_struct
    cs, keep = _cols_struct(c)
    L = _lib.lib()
    L.b2l_serialize_ndjson.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p,
                                       ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                       ctypes.POINTER(ctypes.c_uint64)]
    L.b2l_serialize_free.argtypes = [ctypes.c_void_p]
    out, n = ctypes.c_void_p(), ctypes.c_uint64()
    _lib.check(L.b2l_serialize_ndjson(ctypes.byref(cs), head, len(head), blob, off.ctypes.data,
                                      threads or min(32, os.cpu_count() or 1), ctypes.byref(out), ctypes.byref(n)),
               "b2l_serialize_ndjson")
    del keep
    try:
        return ctypes.string_at(out, n.value)
    finally:
        L.b2l_serialize_free(out)


def serialize_trace(trace, threads: Optional[int] = None) -> bytes:
    """Drop-in for dmlens.traceio.serialize_trace: validate (GPU), refuse invalid traces with
    the reference's InvalidTrace, then the native writer."""
    from .columns import Unrepresentable, to_columns
    from .standalone import validate
    from .types import type_family
    T = type_family(trace)
    violations = validate(trace)
    if trace.version != FORMAT_VERSION:
        violations.append(T.Violation("header", f"version={trace.version} is not serializable as format "
                                                f"{FORMAT_VERSION}"))
    if violations:
        raise _serialize_errors(T)(violations)
    try:
        c = to_columns(trace)
    except Unrepresentable as exc:  # validate() passed, so this cannot happen
        raise _serialize_errors(T)([T.Violation("field-range", str(exc))]) from exc
    return serialize_columns(c, version=trace.version, threads=threads, validate=False)


def write_trace_file(path, trace) -> None:
    """traceio.py:244-246."""
    data = serialize_trace(trace)
    with open(path, "wb") as fh:
        fh.write(data)


# ------------------------------------------------------------------------ exact path (traceio.py:78-191)
def _u64(obj, key, line_no, E):
    value = obj[key]
    if isinstance(value, bool) or not isinstance(value, int):
        raise E(line_no, f'field "{key}" must be an integer, got {value!r}')
    if not 0 <= value <= U64_MAX:
        raise E(line_no, f'field "{key}"={value} outside 64-bit unsigned range')
    return value


def _header_fields(obj, line_no, types):
    """traceio.py:160-172: the header record's checks, in the reference's order."""
    Malformed, Missing, Unsupported, _ = _errors(types)
    if "dmlens" not in obj:
        raise Missing()
    version = obj["dmlens"]
    if version != FORMAT_VERSION:
        raise Unsupported(version)
    nd = _u64(obj, "num_devices", line_no, Malformed)
    host = _u64(obj, "host_device", line_no, Malformed)
    wall = _u64(obj, "wall_time_ns", line_no, Malformed) if "wall_time_ns" in obj else None
    return version, nd, host, wall


def _record_fields(obj, line_no, types):
    """traceio.py:87-151: one event record's checks, in the reference's order -> field dict."""
    Malformed = _errors(types)[0]
    for key in _REQUIRED:
        if key not in obj:
            raise Malformed(line_no, f'missing required field "{key}"')
    kind_str = obj["kind"]
    if kind_str not in _KINDS or not isinstance(kind_str, str):
        raise Malformed(line_no, f"unknown event kind {kind_str!r}")
    t0 = _u64(obj, "t0", line_no, Malformed)
    t1 = _u64(obj, "t1", line_no, Malformed)
    if t1 < t0:
        raise Malformed(line_no, f"event interval inverted (t1 {t1} < t0 {t0})")
    file, ln = obj.get("file"), obj.get("line")
    if file is not None and not isinstance(file, str):
        raise Malformed(line_no, f'field "file" must be a string, got {file!r}')
    if ln is not None and (isinstance(ln, bool) or not isinstance(ln, int) or ln <= 0):
        raise Malformed(line_no, f'field "line" must be a positive integer, got {ln!r}')
    if file is not None and ln is None:
        raise Malformed(line_no, 'field "file" present without "line"')
    codeptr = _u64(obj, "codeptr", line_no, Malformed)
    f = {"seq": _u64(obj, "seq", line_no, Malformed), "kind": kind_str, "t0": t0, "t1": t1,
         "src_dev": _u64(obj, "src_dev", line_no, Malformed), "dst_dev": _u64(obj, "dst_dev", line_no, Malformed),
         "src_addr": _u64(obj, "src_addr", line_no, Malformed), "dst_addr": _u64(obj, "dst_addr", line_no, Malformed),
         "bytes": _u64(obj, "bytes", line_no, Malformed), "hash": _u64(obj, "hash", line_no, Malformed),
         "codeptr": codeptr}
    if file is not None:
        f["file"] = file
    if ln is not None:
        f["line"] = ln
    return f


def _json_object(line: str, line_no: int, types):
    Malformed = _errors(types)[0]
    try:
        obj = json.loads(line)
    except json.JSONDecodeError as exc:
        raise Malformed(line_no, f"invalid JSON: {exc.msg}") from exc
    if not isinstance(obj, dict):
        raise Malformed(line_no, "record is not a JSON object")
    return obj


def _canonical_line(text: str, line_no: int, header: bool, types) -> bytes:
    """One line the native parser could not vouch for, checked as the reference checks it
    (raising its exception), rewritten in the canonical form the native parser reads: blank /
    comment lines (after Python's Unicode-aware strip) become empty, records keep only the
    fields the reference reads."""
    line = text.strip()
    if not line or line.startswith("#"):
        return b""
    obj = _json_object(line, line_no, types)
    if header:
        _, nd, host, wall = _header_fields(obj, line_no, types)
        d = {"dmlens": FORMAT_VERSION, "num_devices": nd, "host_device": host}
        if wall is not None:
            d["wall_time_ns"] = wall
    else:
        d = _record_fields(obj, line_no, types)
    return json.dumps(d, separators=(",", ":"), ensure_ascii=True).encode("ascii")


def _parse_exact(text: str, types=None):
    """Line-by-line restatement of the reference parser (traceio.py:153-191) for traces the
    columns cannot represent: raises its exact exceptions."""
    T = types or family(None)
    Missing = _errors(types)[1]
    Invariant = _errors(types)[3]
    trace, events, cache = None, [], {}
    for line_no, raw in enumerate(text.split("\n"), start=1):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        obj = _json_object(line, line_no, types)
        if trace is None:
            version, nd, host, wall = _header_fields(obj, line_no, types)
            trace = T.Trace(version=version, num_devices_total=nd, host_device=host, wall_time_ns=wall, events=[])
            continue
        f = _record_fields(obj, line_no, types)
        key = (f["codeptr"], f.get("file"), f.get("line"))
        loc = cache.get(key)
        if loc is None:
            loc = cache[key] = T.CodeLocation(codeptr=key[0], file=key[1], line=key[2])
        events.append(T.TraceEvent(
            seq=f["seq"], kind=T.EventKind(f["kind"]), start_ns=f["t0"], end_ns=f["t1"], src_device=f["src_dev"],
            dst_device=f["dst_dev"], src_addr=f["src_addr"], dst_addr=f["dst_addr"], bytes=f["bytes"],
            hash=f["hash"], loc=loc))
    if trace is None:
        raise Missing("empty input: no header line found")
    events.sort(key=lambda e: (e.start_ns, e.seq))
    trace.events = events
    if trace.wall_time_ns is None:
        trace.wall_time_ns = trace.wall_time()
    from .standalone import validate
    violations = validate(trace)
    if violations:
        raise Invariant(violations)
    return trace
