"""paper_2601_12713_b200 -- B200-native engine for the OMPDataPerf hot path
(content hashing of mapped buffers + offline trace analysis), a drop-in
behind the reference analyzer's Python API (dmlens).  See DESIGN.md."""
from __future__ import annotations

__version__ = "0.1.0"

from .errors import (DeviceOutOfRange, EmptyPayload, EngineError, EngineUnavailable,
                     FindingsTraceMismatch, InvalidTrace)
from .hashing import (CollisionAuditStore, HashFn, audit_observe, hash_batch, hash_bytes, hash_device,
                      hash_tensors, make_hasher)
from .analysis import (ColumnarFindings, ColumnarSavings, analyze, analyze_columns, analyze_many, attribute,
                       estimate, savings_columns)
from .columns import Columns, columns_from_arrays, to_columns
from . import ingest, multigpu, reporting, sharded, synth  # noqa: F401  (submodules of the public API)
from .standalone import (find_duplicate_transfers, find_repeated_allocs, find_round_trips, find_unused_allocs,
                         find_unused_transfers, get_alloc_delete_pairs, sort_by_device, validate)

__all__ = [
    "DeviceOutOfRange", "EmptyPayload", "EngineError", "EngineUnavailable",
    "FindingsTraceMismatch", "InvalidTrace", "HashFn", "hash_batch", "hash_bytes",
    "hash_device", "hash_tensors", "make_hasher", "CollisionAuditStore", "audit_observe", "ColumnarFindings", "ColumnarSavings", "analyze",
    "analyze_columns", "analyze_many", "attribute", "estimate", "savings_columns", "Columns", "columns_from_arrays", "to_columns",
    "find_duplicate_transfers", "find_repeated_allocs", "find_round_trips", "find_unused_allocs",
    "find_unused_transfers", "get_alloc_delete_pairs", "sort_by_device", "validate",
]
