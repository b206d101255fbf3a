"""CPU: libb2l.so loads and exports every symbol include/b2l.h declares
(no compute calls -- there is no GPU here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "b2l.h")).read()
    # function declarations: "<type> [*]b2l_name(" at the start of a line
    return sorted(set(re.findall(r"^(?:int|int32_t|void|const char \*|b2l_capture \*)\s*\*?(b2l_[a-z0-9_]+)\(", src, re.M)))


def test_library_exports_header_symbols():
    from paper_2601_12713_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert "b2l_hash_batch" in syms
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED) <= set(syms)


def test_abi_version_and_no_device_error():
    from paper_2601_12713_b200 import _lib
    assert _lib.lib().b2l_abi_version() == 1
    # no GPU in this container: the device count call must fail cleanly, not crash
    n = _lib.device_count()
    assert n >= 0


def test_hash_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        import pytest
        pytest.skip("device present")
    import pytest
    from paper_2601_12713_b200 import EngineError, hash_bytes
    with pytest.raises(EngineError):
        hash_bytes(b"abc")


def test_hash_large_many_argument_errors():
    """b2l_hash_large_many checks its arguments before touching a device (hashing.py:29 maps a
    zero-length payload to EmptyPayload; null arrays are B2L_E_INVALID_ARG)."""
    import numpy as np
    import pytest
    from paper_2601_12713_b200 import _lib
    from paper_2601_12713_b200.errors import EmptyPayload
    from paper_2601_12713_b200.hashing import hash_large_many
    L = _lib.lib()
    assert L.b2l_hash_large_many(None, None, 0, None, None) == 0  # nothing to hash
    assert L.b2l_hash_large_many(None, None, 1, None, None) != 0
    ptrs = np.array([4096, 8192], dtype=np.uint64)
    lens = np.array([16, 0], dtype=np.uint64)
    assert L.b2l_hash_large_many(ptrs.ctypes.data, lens.ctypes.data, 2, 64, None) != 0
    assert b"zero-byte" in L.b2l_last_error()
    with pytest.raises(EmptyPayload):
        hash_large_many([4096, 8192], [16, 0], 64)
