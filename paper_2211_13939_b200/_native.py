"""ctypes binding of ``libincrtts_b200.so`` (C ABI: ``include/incrtts_b200.h``).

The library is built in-tree by ``_build.py`` (``__graft_entry__.build()``).
There is deliberately no fallback: if the library is missing or fails to
load, every GPU module raises here -- the product path never degrades to a
CPU or eager-PyTorch implementation.
"""

from __future__ import annotations

import ctypes
import os
import re
from functools import lru_cache
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libincrtts_b200.so"
HEADER = PKG.parent / "include" / "incrtts_b200.h"

_i32, _i64, _f64, _p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
_ERRORS = {10001: "ITTS_EINVAL", 10002: "ITTS_EALIGN", 10003: "ITTS_EUNSUPPORTED"}

# name -> argtypes (all return int status)
SIGNATURES: dict[str, list] = {
    "itts_version": [],
    "itts_gather_rows": [_p, _p, _i32, _i64, _p],
    "itts_scatter_rows": [_p, _p, _i32, _i64, _p],
    "itts_s_encode": [_p, _i64, _p, _i32, _i64, _i32, _p, _p],
    "itts_s_decode_chunk": [_p, _i32, _i32, _f64, _p],
    "itts_s_vocode_chunk": [_p, _i32, _i32, _i32, _i32, _i64, _p, _p, _p],
    "itts_conv1d_tc": [_p, _i64, _i32, _i64, _p, _i32, _i32, _p, _p, _i32, _p, _p, ctypes.c_float, _p, _i32,
                       _p, _i32, _p, ctypes.c_float, _i32, _i32, _p],
    "itts_resblock_tc": [_p, _i64, _i32, _p, _p, _p, _p, _i32, _i32, _p, _p, _i32, _p, ctypes.c_float, _p],
    "itts_resblock_debug_trace": [_p],
    "itts_r_dec_prepare": [_p, _p, _i32, _p],
    "itts_r_decode_debug_trace": [_p],
    "itts_r_decode_persistent": [_i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                                 _p, _p, _p, _i64, _p, _p, _p, _p, _i32, _p],
    "itts_r_prenet": [_p, _p, _p, _p, _p, _p, _i32, _i32, _p],
    "itts_r_lstm_cell": [_p, _i32, _p, _p, _p, _i32, _i32, _p, _i32, _i32, _p],
    "itts_r_query": [_p, _p, _p, _i32, _p],
    "itts_r_attention": [_p, _p, _p, _i32, _i32, _p, _p, _p, _p, _i32, _p],
    "itts_r_proj": [_p, _p, _i32, _p, _p, _p, _i32, _p],
    "itts_r_enc_embed": [_p, _i64, _p, _i32, _i64, _p, _p, _p, _p, _p, _p],
    "itts_r_bilstm": [_p, _p, _i32, _p, _p],
    "itts_r_bilstm_tc": [_p, _p, _i32, _p, _p],
    "itts_r_pmem": [_p, _i32, _i64, _p, _p],
    "itts_r_mel_assemble": [_p, _i32, _i64, _p, _i32, _p],
    "itts_r_rowmap": [_p, _i32, _i64, _p, _p],
    "itts_r_zero_halo": [_p, _i32, _i64, _p, _i32, _p],
    "itts_r_encode": [_p, _i64, _i32, _i64, _i64, _i64, _p, _i32, _p, _p, _p, _p, _p],
    "itts_r_encode_split": [_p, _i64, _i32, _i64, _i64, _i64, _p, _i32, _p, _p, _p, _p, _i32, _p],
    "itts_bert_prosody": [_p, _p, _p, _i32, _i64, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "itts_r_postnet": [_p, _i32, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _p],
    "itts_r_mrf_combine": [_p, _p, _p, _i64, ctypes.c_float, _p, _p],
    "itts_r_voc_create": [_p, _p, _i32],
    "itts_r_voc_reserve": [_p, _i32, _i32, _p],
    "itts_r_voc_run": [_p, _i32, _p, _p, _i32, _p, _p],
    "itts_r_voc_destroy": [_p],
    "itts_r_pcm16_b64": [_p, _p, _i32, _i64, _p, _p],
    "itts_r_post_splice": [_p, _p, _i32, _i64, _p, ctypes.c_float, _p, _i32, _i32, _p, _p, _p, _p],
}


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


def header_symbols() -> list[str]:
    """Every ``itts_*`` function the public header declares."""
    return sorted(set(re.findall(r"\bint\s+(itts_\w+)\s*\(", HEADER.read_text())))


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    # ITTS_LIB: an alternative build of the same library (A/B timing tools only)
    path = Path(os.environ.get("ITTS_LIB", LIB_PATH))
    if not path.exists():
        raise NativeError(f"{path} is missing: run __graft_entry__.build() "
                          "(no CPU fallback exists for the GPU modules)")
    handle = ctypes.CDLL(str(path))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    return handle


def call(name: str, *args) -> None:
    status = getattr(lib(), name)(*args)
    if status != 0:
        what = _ERRORS.get(status, f"cudaError {status}")
        raise NativeError(f"{name} failed: {what}")
