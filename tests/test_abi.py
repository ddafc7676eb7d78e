"""The C-ABI library loads without a GPU and exports every symbol include/b2s.h declares."""

import ctypes

from paper_2602_08387_b200 import _lib


def test_library_exports_declared_symbols():
    lib = _lib.load()
    declared = _lib.declared_symbols()
    assert "b2s_gather_samples" in declared
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.b2s_abi_version() >= 1


def test_error_reporting():
    lib = _lib.load()
    w = ctypes.c_int()
    assert lib.b2s_token_width_for_vocab(0, ctypes.byref(w)) == _lib.B2S_EINVAL
    assert "vocab_size" in _lib.last_error()
