"""Host-side record types of the drop-in API.

Field names, order and semantics mirror the reference's public types so the
engine's results compare equal to the reference's (and are the reference's
own classes when the input trace is a ``dmlens`` trace -- see ``type_family``):

  EventKind, CodeLocation, TraceEvent, Trace, Violation  dmlens/model.py:29-117
  AllocPair, PrepWarning                                 dmlens/prep.py:19-32
  DuplicateGroup, RoundTripGroup, RepeatedAllocGroup,
  Findings                                               dmlens/detectors.py:33-76
  SavingsEstimate                                        dmlens/estimator.py:41-48
  AttributedIssue                                        dmlens/report.py:34-41

These are plain containers; all analysis arithmetic runs in libb2l.so.
"""
from __future__ import annotations

import sys
from dataclasses import dataclass, field
from enum import Enum
from types import SimpleNamespace
from typing import Optional


class EventKind(Enum):
    TRANSFER = "transfer"
    ALLOC = "alloc"
    DELETE = "delete"
    KERNEL = "kernel"


KIND_CODE = {"transfer": 0, "alloc": 1, "delete": 2, "kernel": 3}  # column encoding (include/b2l.h)


@dataclass(slots=True)
class CodeLocation:
    codeptr: int = 0
    file: Optional[str] = None
    line: Optional[int] = None


@dataclass(slots=True)
class TraceEvent:
    seq: int
    kind: EventKind
    start_ns: int
    end_ns: int
    src_device: int
    dst_device: int
    src_addr: int
    dst_addr: int
    bytes: int
    hash: int
    loc: CodeLocation = field(default_factory=CodeLocation)

    def duration_ns(self) -> int:
        return self.end_ns - self.start_ns


@dataclass(slots=True)
class Trace:
    version: int
    num_devices_total: int
    host_device: int
    wall_time_ns: Optional[int]
    events: list

    def wall_time(self) -> int:
        if self.wall_time_ns is not None:
            return self.wall_time_ns
        if not self.events:
            return 0
        return max(e.end_ns for e in self.events) - min(e.start_ns for e in self.events)

    def target_devices(self):
        return (d for d in range(self.num_devices_total) if d != self.host_device)


@dataclass(slots=True)
class Violation:
    rule: str
    message: str
    seq: Optional[int] = None

    def __str__(self) -> str:
        where = f" (seq {self.seq})" if self.seq is not None else ""
        return f"{self.rule}: {self.message}{where}"


@dataclass(slots=True)
class AllocPair:
    alloc_event: TraceEvent
    delete_event: TraceEvent
    synthetic_delete: bool = False


@dataclass(slots=True)
class PrepWarning:
    seq: int
    reason: str

    def __str__(self) -> str:
        return f"seq {self.seq}: {self.reason}"


@dataclass(slots=True)
class DuplicateGroup:
    hash: int
    dest_device: int
    events: list


@dataclass(slots=True)
class RoundTripGroup:
    hash: int
    src_device: int
    dest_device: int
    trips: list


@dataclass(slots=True)
class RepeatedAllocGroup:
    host_addr: int
    tgt_device: int
    bytes: int
    pairs: list


@dataclass(slots=True)
class Findings:
    duplicates: list = field(default_factory=list)
    round_trips: list = field(default_factory=list)
    repeated_allocs: list = field(default_factory=list)
    unused_allocs: list = field(default_factory=list)
    unused_transfers: list = field(default_factory=list)

    def total_count(self) -> int:
        return (len(self.duplicates) + len(self.round_trips) + len(self.repeated_allocs)
                + len(self.unused_allocs) + len(self.unused_transfers))


@dataclass(slots=True)
class SavingsEstimate:
    per_category_ns: dict
    union_ns: int
    wall_time_ns: int
    predicted_speedup: float
    eliminable_seqs: frozenset
    warnings: tuple


@dataclass(slots=True)
class AttributedIssue:
    category: str
    location: CodeLocation
    occurrence_count: int
    total_ns: int
    total_bytes: int
    pct_of_wall: float


_OWN = SimpleNamespace(
    EventKind=EventKind, CodeLocation=CodeLocation, TraceEvent=TraceEvent, Trace=Trace, Violation=Violation,
    AllocPair=AllocPair, PrepWarning=PrepWarning, DuplicateGroup=DuplicateGroup, RoundTripGroup=RoundTripGroup,
    RepeatedAllocGroup=RepeatedAllocGroup, Findings=Findings, SavingsEstimate=SavingsEstimate,
    AttributedIssue=AttributedIssue, InvalidTrace=None, FindingsTraceMismatch=None, root=None)


def type_family(obj) -> SimpleNamespace:
    """The result classes to build for an input trace: the reference's own
    (dmlens.*) when the trace came from dmlens, so results compare equal and
    isinstance() checks in reference code keep working; ours otherwise."""
    mod = type(obj).__module__
    if mod.startswith("dmlens"):
        return family(mod.split(".")[0])
    return _OWN


def family(root: str = None) -> SimpleNamespace:
    """Class family by package name: None -> ours, "dmlens" -> the reference's."""
    if root is None:
        return _OWN
    import importlib
    m = importlib.import_module(root + ".model")
    d = importlib.import_module(root + ".detectors")
    p = importlib.import_module(root + ".prep")
    e = importlib.import_module(root + ".estimator")
    r = importlib.import_module(root + ".report")
    return SimpleNamespace(
        EventKind=m.EventKind, CodeLocation=m.CodeLocation, TraceEvent=m.TraceEvent, Trace=m.Trace,
        Violation=m.Violation, AllocPair=p.AllocPair, PrepWarning=p.PrepWarning,
        DuplicateGroup=d.DuplicateGroup, RoundTripGroup=d.RoundTripGroup,
        RepeatedAllocGroup=d.RepeatedAllocGroup, Findings=d.Findings, SavingsEstimate=e.SavingsEstimate,
        AttributedIssue=r.AttributedIssue, InvalidTrace=d.InvalidTrace,
        FindingsTraceMismatch=e.FindingsTraceMismatch, root=root)
