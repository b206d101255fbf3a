"""Exception types of the engine; names and messages follow the reference's
(dmlens.hashing.EmptyPayload hashing.py:29-31, dmlens.detectors.InvalidTrace
detectors.py:79-82, dmlens.prep.DeviceOutOfRange prep.py:35-39,
dmlens.estimator.FindingsTraceMismatch estimator.py:35-38)."""
from __future__ import annotations


class EngineError(RuntimeError):
    """A CUDA / engine failure reported through the C ABI."""


class EngineUnavailable(EngineError):
    """libb2l.so is not built or no CUDA device is present: there is no fallback."""


class EmptyPayload(ValueError):
    def __init__(self) -> None:
        super().__init__("cannot hash a zero-byte payload")


class InvalidTrace(Exception):
    def __init__(self, violations):
        super().__init__(f"trace fails validation with {len(violations)} violations")
        self.violations = violations


class DeviceOutOfRange(Exception):
    def __init__(self, seq: int, device: int, num_devices_total: int):
        super().__init__(f"event seq {seq}: device {device} outside [0, {num_devices_total})")
        self.seq = seq
        self.device = device


class FindingsTraceMismatch(Exception):
    def __init__(self, seq: int):
        super().__init__(f"findings reference event seq {seq} absent from the trace")
        self.seq = seq
