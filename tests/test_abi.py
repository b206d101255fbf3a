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
