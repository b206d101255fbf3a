"""ctypes binding of libb2l.so (the C ABI in include/b2l.h).

The product path has no CPU fallback: if the shared library is missing or
cannot be loaded, every entry point raises ``EngineUnavailable``.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import (DeviceOutOfRange, EmptyPayload, EngineError, EngineUnavailable,
                     FindingsTraceMismatch, InvalidTrace)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libb2l.so")

B2L_OK = 0
B2L_E_INVALID_ARG = -1
B2L_E_EMPTY_PAYLOAD = -2
B2L_E_INVALID_TRACE = -3
B2L_E_DEVICE_RANGE = -4
B2L_E_CUDA = -5
B2L_E_OOM = -6
B2L_E_MISMATCH = -7
B2L_E_NO_DEVICE = -8

# every symbol include/b2l.h declares (tests check the library exports all of them)
EXPORTED = (
    "b2l_abi_version", "b2l_last_error", "b2l_device_count",
    "b2l_hash_batch", "b2l_hash_host", "b2l_hash_bytes", "b2l_fill_payloads",
    "b2l_hash_launch_info", "b2l_hash_select_variant", "b2l_hash_large", "b2l_hash_large_many",
    "b2l_analyze", "b2l_analyze_ex", "b2l_findings_free", "b2l_savings_compute", "b2l_savings_free",
    "b2l_lookup_seqs", "b2l_audit_batch", "b2l_stable_sort_u32", "b2l_stable_sort_u64", "b2l_shard_route", "b2l_shard_unpack", "b2l_sort_u64_pairs_device",
    "b2l_shard_kernel_summary", "b2l_shard_route_pairs",
    "b2l_capture_create", "b2l_capture_destroy", "b2l_capture_set_audit_dir", "b2l_capture_device_slot",
    "b2l_capture_target", "b2l_capture_data_op", "b2l_capture_finalize", "b2l_capture_free_text",
    "b2l_capture_write", "b2l_capture_warnings",
    "b2l_init", "b2l_shutdown", "b2l_ngpus", "b2l_lpt_partition", "b2l_hash_host_multi",
    "b2l_serialize_ndjson", "b2l_serialize_free", "b2l_ingest_ndjson", "b2l_ingest_free",
)

_u64 = ctypes.c_uint64
_p = ctypes.c_void_p
_pu64 = ctypes.POINTER(ctypes.c_uint64)
_int = ctypes.c_int

_lock = threading.Lock()
_lib = None


def _declare(lib):
    sig = {
        "b2l_abi_version": ([], _int),
        "b2l_last_error": ([], ctypes.c_char_p),
        "b2l_device_count": ([ctypes.POINTER(_int)], _int),
        "b2l_hash_batch": ([_p, _p, _u64, _p, _p, _p], _int),
        "b2l_hash_host": ([_p, _p, _u64, _p], _int),
        "b2l_hash_bytes": ([_p, _u64, _pu64], _int),
        "b2l_fill_payloads": ([_p, _p, _p, _p, _u64, _u64, _p], _int),
        "b2l_hash_select_variant": ([_int, ctypes.POINTER(_int)], _int),
        "b2l_hash_large": ([_p, _u64, _p, _p], _int),
        "b2l_hash_large_many": ([_p, _p, _u64, _p, _p], _int),
        "b2l_hash_launch_info": ([_u64, ctypes.POINTER(_int), ctypes.POINTER(_int), ctypes.POINTER(_int)], _int),
        "b2l_init": ([_int, ctypes.POINTER(_int)], _int),
        "b2l_shutdown": ([], _int),
        "b2l_ngpus": ([ctypes.POINTER(_int), ctypes.POINTER(_int), _int], _int),
        "b2l_lpt_partition": ([_p, _u64, ctypes.c_uint32, _p, _p], _int),
        "b2l_hash_host_multi": ([_p, _p, _u64, _p], _int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def lib():
    """The loaded engine library (raises EngineUnavailable if it is not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise EngineUnavailable(
                        f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
                try:
                    _lib = _declare(ctypes.CDLL(LIB_PATH))
                except OSError as exc:  # pragma: no cover - depends on the box
                    raise EngineUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    return _lib


def last_error() -> str:
    msg = lib().b2l_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a B2L_E_* return code to the reference's exception classes."""
    if rc == B2L_OK:
        return
    msg = last_error()
    if rc == B2L_E_EMPTY_PAYLOAD:
        raise EmptyPayload()
    if rc == B2L_E_MISMATCH:
        raise FindingsTraceMismatch(-1)
    if rc in (B2L_E_CUDA, B2L_E_OOM, B2L_E_NO_DEVICE):
        raise EngineUnavailable(f"{what}: {msg}") if rc == B2L_E_NO_DEVICE else EngineError(f"{what}: {msg}")
    raise EngineError(f"{what}: code {rc}: {msg}")


def device_count() -> int:
    n = _int(0)
    rc = lib().b2l_device_count(ctypes.byref(n))
    return n.value if rc == B2L_OK else 0


__all__ = ["lib", "check", "last_error", "device_count", "EXPORTED", "LIB_PATH",
           "InvalidTrace", "DeviceOutOfRange"]
