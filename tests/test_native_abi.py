"""The C-ABI library loads and exports every symbol the public header declares (CPU-only)."""

import ctypes

import pytest

from paper_2211_13939_b200 import _native


def test_library_exports_header_symbols():
    lib = _native.lib()
    declared = _native.header_symbols()
    assert declared, "header declares no itts_* functions"
    missing = [name for name in declared if not hasattr(lib, name)]
    assert not missing, missing
    assert set(declared) == set(_native.SIGNATURES), "ctypes table out of sync with the header"


def test_version_and_argument_errors_need_no_gpu():
    lib = _native.lib()
    assert lib.itts_version() >= 1
    # argument validation happens before any CUDA call, so it works without a device
    assert lib.itts_gather_rows(None, None, 1, 16, None) == 10001
    assert lib.itts_gather_rows(ctypes.c_void_p(8), ctypes.c_void_p(16), 1, 24, None) == 10002
    assert lib.itts_s_decode_chunk(None, 0, 8, 0.1, None) == 0
    assert lib.itts_s_decode_chunk(ctypes.c_void_p(16), 1, 7, 0.1, None) == 10003
    with pytest.raises(_native.NativeError, match="ITTS_EINVAL"):
        _native.call("itts_scatter_rows", None, None, 2, 16, None)
