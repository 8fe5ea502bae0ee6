"""ctypes binding of libeq4.so (include/eq4.h).

The library is the product: there is no Python or CPU fallback.  If the
shared object is missing or no CUDA device is present, every entry point
raises instead of computing something else.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EQ4_LIB") or os.path.join(HERE, "libeq4.so")

EQ4_OK = 0
EQ4_EINVAL = 1
EQ4_ECUDA = 2
EQ4_EDATA = 3
EQ4_ERANGE = 4
EQ4_EUNSUPPORTED = 5

METHOD = {"asym": 0, "greedy": 1, "hist-brute": 2, "sym": 3, "aciq": 4, "gss": 5, "table": 6,
          "hist-apprx": 7}
AUX = {"fp32": 0, "fp16": 1}
STATUS_NONFINITE = 1
STATUS_RANGE = 2
STATUS_QUERY = 4
STATUS_INDEX = 8

# every symbol include/eq4.h declares (tests check the .so exports them all)
EXPORTS = (
    "eq4_version",
    "eq4_last_error",
    "eq4_packed_row_stride",
    "eq4_quantize_pack",
    "eq4_quantize_pack_p",
    "eq4_row_range_f64",
    "eq4_quantize_pack_host",
    "eq4_pack",
    "eq4_unpack",
    "eq4_quant_mse",
    "eq4_sparse_lengths_sum4",
    "eq4_kmeans_row_stride",
    "eq4_kmeans_rows",
    "eq4_quantize_file",
    "eq4_write_embq",
    "eq4_selftest",
    "eq4_diag_counters",
    "eq4_quantize_rows",
    "eq4_dequantize_rows",
    "eq4_build_histogram",
    "eq4_bin_l2_norm",
    "eq4_quant_mse_rows",
)

_lib = None
_lock = threading.Lock()


class Eq4Error(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load libeq4.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise Eq4Error(
                f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; g.build()\"`"
                " (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.eq4_version.restype = ctypes.c_char_p
        L.eq4_last_error.restype = ctypes.c_char_p
        L.eq4_packed_row_stride.argtypes = [i64, i32]
        L.eq4_packed_row_stride.restype = i64
        L.eq4_quantize_pack.argtypes = [vp, i64, i64, i64, i32, i32, dbl, i32, vp, vp, vp, vp, vp,
                                        vp, vp, vp]
        L.eq4_quantize_pack.restype = i32
        L.eq4_quantize_pack_p.argtypes = [vp, i64, i64, i64, i32, i32, dbl, dbl, i32, vp, vp, vp, vp,
                                          vp, vp, vp, vp]
        L.eq4_quantize_pack_p.restype = i32
        L.eq4_row_range_f64.argtypes = [vp, i64, i64, i64, i32, dbl, vp, vp, vp, vp, vp]
        L.eq4_row_range_f64.restype = i32
        L.eq4_quantize_pack_host.argtypes = [vp, i64, i64, i64, i32, i32, dbl, i32, vp, vp, vp, vp,
                                             vp, vp, i64, vp, vp]
        L.eq4_quantize_pack_host.restype = i32
        L.eq4_pack.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp]
        L.eq4_pack.restype = i32
        L.eq4_unpack.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp]
        L.eq4_unpack.restype = i32
        L.eq4_quant_mse.argtypes = [vp, i64, i64, i64, vp, vp, vp, vp]
        L.eq4_quant_mse.restype = i32
        L.eq4_sparse_lengths_sum4.argtypes = [vp, i64, i64, i32, vp, i64, vp, i64, vp, vp, vp, vp]
        L.eq4_sparse_lengths_sum4.restype = i32
        L.eq4_kmeans_row_stride.argtypes = [i64, i32]
        L.eq4_kmeans_row_stride.restype = i64
        L.eq4_kmeans_rows.argtypes = [vp, i64, i64, i64, i32, vp, vp, vp, vp]
        L.eq4_kmeans_rows.restype = i32
        cp = ctypes.c_char_p
        L.eq4_quantize_file.argtypes = [cp, cp, i32, i32, dbl, i32, i64, vp, vp]
        L.eq4_quantize_file.restype = i32
        L.eq4_write_embq.argtypes = [cp, vp, i64, i64, i32, i32]
        L.eq4_write_embq.restype = i32
        L.eq4_selftest.argtypes = [i32, i64, ctypes.c_uint64]
        L.eq4_selftest.restype = ctypes.c_longlong
        L.eq4_diag_counters.argtypes = [vp, i32]
        L.eq4_diag_counters.restype = i32
        L.eq4_quantize_rows.argtypes = [vp, i32, i64, i64, i64, vp, vp, i64, i32, i32, vp, vp, vp, vp]
        L.eq4_quantize_rows.restype = i32
        L.eq4_dequantize_rows.argtypes = [vp, i64, i64, vp, vp, i32, vp, vp]
        L.eq4_dequantize_rows.restype = i32
        L.eq4_build_histogram.argtypes = [vp, i32, i64, i64, i64, i32, vp, vp, vp, vp]
        L.eq4_build_histogram.restype = i32
        L.eq4_bin_l2_norm.argtypes = [vp, vp, vp, i64, vp, vp]
        L.eq4_bin_l2_norm.restype = i32
        L.eq4_quant_mse_rows.argtypes = [vp, i32, i64, i64, i64, vp, vp, i32, vp, vp]
        L.eq4_quant_mse_rows.restype = i32
        _lib = L
    return _lib


def last_error() -> str:
    return load().eq4_last_error().decode()


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == EQ4_OK:
        return
    msg = last_error()
    if rc in (EQ4_EINVAL, EQ4_EDATA, EQ4_ERANGE, EQ4_EUNSUPPORTED):
        raise ValueError(msg)
    raise Eq4Error(msg)


def packed_row_stride(dim: int, aux: str) -> int:
    return int(load().eq4_packed_row_stride(int(dim), AUX[aux]))


def diag_counters(reset: bool = False) -> dict:
    """GREEDY rare-path counters of the current device (eq4_diag_counters)."""
    import numpy as np

    out = np.zeros(5, np.int64)
    check(load().eq4_diag_counters(out.ctypes.data_as(ctypes.c_void_p), int(bool(reset))))
    return {"exact_redecisions": int(out[0]), "exact_code_rows": int(out[1]),
            "near_count_checks": int(out[2]), "near_count_escalations": int(out[3]),
            "deferred_rows": int(out[4])}
