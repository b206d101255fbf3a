"""Capture agent: the reference's capture shim model (pkg/shim/src/capture.ts:93-327, SPEC.md
"ompt-shim") over the native agent in libb2l (b2l_capture_*), with transfer payloads hashed on
the GPU where they live -- the landed device copy of a host-to-device transfer, the device
source of a device-to-host one -- and host buffers only when nothing else is offered.

The native OMPT tool (libb2l_ompt.so: ompt_start_tool + the target / target-data-op EMI
callbacks) drives the same agent inside an OpenMP program; this class is the library surface
(and what the tests drive, as capture.test.ts drives CaptureShim)."""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

from . import _lib

BEGIN, END = 1, 2
OPTYPES = {"alloc": 1, "transfer_to_device": 2, "transfer_from_device": 3, "delete": 4}
_NOW = 2**64 - 1


@dataclass
class ShimWarnings:
    unmatched_ends: int
    unfinished_at_exit: int
    hash_skipped: int
    dropped_malformed: int


def _L():
    L = _lib.lib()
    L.b2l_capture_create.restype = ctypes.c_void_p
    L.b2l_capture_create.argtypes = [ctypes.c_int32]
    L.b2l_capture_destroy.argtypes = [ctypes.c_void_p]
    L.b2l_capture_set_audit_dir.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
    L.b2l_capture_device_slot.argtypes = [ctypes.c_void_p, ctypes.c_int32]
    L.b2l_capture_device_slot.restype = ctypes.c_int32
    L.b2l_capture_target.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int32,
                                     ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
    L.b2l_capture_data_op.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                      ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_void_p]
    L.b2l_capture_finalize.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p),
                                       ctypes.POINTER(ctypes.c_uint64)]
    L.b2l_capture_free_text.argtypes = [ctypes.c_void_p]
    L.b2l_capture_write.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_uint64]
    L.b2l_capture_warnings.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
    return L


def _ptr(buf):
    """(address, keep-alive) of a payload view: a torch CUDA tensor (device), a torch CPU tensor,
    bytes / bytearray / memoryview / numpy array (host)."""
    if buf is None:
        return None, None
    if hasattr(buf, "data_ptr"):
        return buf.data_ptr(), buf
    import numpy as np
    a = np.frombuffer(bytes(buf), dtype=np.uint8) if isinstance(buf, (bytes, memoryview)) else np.ascontiguousarray(buf)
    return a.ctypes.data, a


class CaptureShim:
    """CaptureShim(host_device_id, out_path=None, audit_dir=None, clock=None) -- capture.ts:93-121."""

    host_slot = 0

    def __init__(self, host_device_id: int, out_path: Optional[str] = None, audit_dir: Optional[str] = None,
                 clock=None):
        self._L = _L()
        self._c = self._L.b2l_capture_create(int(host_device_id))
        if not self._c:
            raise MemoryError(_lib.last_error())
        self.out_path, self.clock = out_path, clock
        audit = audit_dir if audit_dir is not None else os.environ.get("DMLENS_AUDIT_DIR")
        _lib.check(self._L.b2l_capture_set_audit_dir(self._c, audit.encode() if audit else None), "audit dir")

    def __del__(self):
        if getattr(self, "_c", None):
            self._L.b2l_capture_destroy(self._c)
            self._c = None

    def _t(self, t):
        if t is not None:
            return int(t)
        return int(self.clock()) if self.clock else _NOW

    def device_slot(self, runtime_id: int) -> int:
        return int(self._L.b2l_capture_device_slot(self._c, int(runtime_id)))

    @property
    def warnings(self) -> ShimWarnings:
        w = (ctypes.c_uint64 * 4)()
        _lib.check(self._L.b2l_capture_warnings(self._c, w), "b2l_capture_warnings")
        return ShimWarnings(*[int(x) for x in w])

    # -- target (kernel) callbacks: capture.ts:164-189
    def on_target_begin(self, target_id, device_id, codeptr=0, thread_id=0, time_ns=None):
        _lib.check(self._L.b2l_capture_target(self._c, BEGIN, int(target_id), int(device_id), int(codeptr),
                                              int(thread_id), self._t(time_ns)), "b2l_capture_target")

    def on_target_end(self, target_id, device_id=0, codeptr=0, thread_id=0, time_ns=None):
        _lib.check(self._L.b2l_capture_target(self._c, END, int(target_id), int(device_id), int(codeptr),
                                              int(thread_id), self._t(time_ns)), "b2l_capture_target")

    # -- data-op callbacks: capture.ts:193-275.  device_buffer: the device copy (torch CUDA tensor
    # or address); host_buffer: the host-side bytes, when that is what the runtime offers
    def _op(self, ep, host_op_id, optype, src_device_id, dest_device_id, src_addr, dest_addr, bytes_, codeptr,
            thread_id, time_ns, device_buffer, host_buffer):
        dptr, dkeep = (device_buffer, None) if isinstance(device_buffer, int) else _ptr(device_buffer)
        hptr, hkeep = _ptr(host_buffer)
        _lib.check(self._L.b2l_capture_data_op(self._c, ep, int(host_op_id), OPTYPES[optype], int(src_device_id),
                                               int(dest_device_id), int(src_addr or 0), int(dest_addr or 0),
                                               int(bytes_ or 0), int(codeptr or 0), int(thread_id),
                                               self._t(time_ns), dptr, hptr), "b2l_capture_data_op")
        del dkeep, hkeep

    def on_data_op_begin(self, host_op_id, optype, src_device_id, dest_device_id, src_addr=0, dest_addr=0,
                         bytes=0, codeptr=0, thread_id=0, time_ns=None, device_buffer=None, host_buffer=None):
        self._op(BEGIN, host_op_id, optype, src_device_id, dest_device_id, src_addr, dest_addr, bytes, codeptr,
                 thread_id, time_ns, device_buffer, host_buffer)

    def on_data_op_end(self, host_op_id, optype, src_device_id, dest_device_id, src_addr=0, dest_addr=0,
                       bytes=0, codeptr=0, thread_id=0, time_ns=None, device_buffer=None, host_buffer=None):
        self._op(END, host_op_id, optype, src_device_id, dest_device_id, src_addr, dest_addr, bytes, codeptr,
                 thread_id, time_ns, device_buffer, host_buffer)

    # -- finalize / writeTrace: capture.ts:279-321
    def finalize(self, wall_time_ns: Optional[int] = None) -> str:
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        _lib.check(self._L.b2l_capture_finalize(self._c, _NOW if wall_time_ns is None else int(wall_time_ns),
                                                ctypes.byref(p), ctypes.byref(n)), "b2l_capture_finalize")
        try:
            return ctypes.string_at(p, n.value).decode()
        finally:
            self._L.b2l_capture_free_text(p)

    def write_trace(self, wall_time_ns: Optional[int] = None) -> str:
        path = self.out_path if self.out_path is not None else os.environ.get("DMLENS_OUT")
        _lib.check(self._L.b2l_capture_write(self._c, path.encode() if path else None,
                                             _NOW if wall_time_ns is None else int(wall_time_ns)),
                   "b2l_capture_write")
        return path
