"""CPU oracle for the row-wise 4-bit clip-search + pack path -- TEST INFRASTRUCTURE.

This package restates the reference (`embquant`, /root/reference/pkg/src) for
the hot path in plain C (``eq4_oracle.c``) plus a numpy port of its seeded
table generator (``rng.py``).  It exists to *check* the CUDA product path and
to time the reference algorithm on the host CPU (bench.py's ``cpu_baseline``
and ``--impl reference`` legs).  Nothing in ``paper_1911_02079_b200`` imports
it; the product path fails loudly when its CUDA library is missing instead of
falling back here.

Pinned against the reference itself: tests/golden/*.npz were produced by
tests/golden/make_golden.py, which imports the real reference in the build
container; tests/test_oracle_golden.py checks this oracle bit-for-bit against
them (HIST-BRUTE: identical window selection, see eq4_oracle.c header).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libeq4_oracle.so")
_lib = None

METHODS = {"asym": 0, "greedy": 1, "hist-brute": 2, "sym": 3, "aciq": 4, "gss": 5, "table": 6,
           "hist-apprx": 7}
AUX = {"fp32": 0, "fp16": 1}

ERRORS = {
    1: "b must be >= 1",
    2: "r must be in (0, 1]",
    3: "input vector is empty",
    4: "invalid clip range",
    5: "table contains non-finite values (NaN/Inf)",
    6: "nbits must be 4 or 8",
    7: "allocation failed",
    8: "unknown method",
    9: "lengths must be non-negative",
    10: "lengths do not sum to the number of indices",
    11: "query index out of range",
}


class OracleError(ValueError):
    def __init__(self, code: int):
        super().__init__(f"oracle error {code}: {ERRORS.get(code, '?')}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile the oracle shared library (make -C oracle)."""
    src = os.path.join(_HERE, "eq4_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_long, ctypes.c_int, ctypes.c_double
        L.eqo_np_sum.argtypes = [vp, i64]
        L.eqo_np_sum.restype = dbl
        L.eqo_quant_mse.argtypes = [vp, i64, dbl, dbl, i32, vp, vp]
        L.eqo_clip_range_greedy.argtypes = [vp, i64, i32, i32, dbl, vp, vp, vp, vp, vp, vp]
        L.eqo_build_histogram.argtypes = [vp, i64, i32, vp, vp, vp]
        L.eqo_bin_l2_norm.argtypes = [dbl, dbl, dbl]
        L.eqo_bin_l2_norm.restype = dbl
        L.eqo_offset_unit_norms.argtypes = [vp, i64, dbl, dbl, vp]
        L.eqo_hist_brute.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.eqo_kmeans_table.argtypes = [vp, i64, i64, i64, i32, vp, vp, vp, i32]
        L.eqo_hist_apprx.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.eqo_hist_apprx_gap.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, vp, vp]
        L.eqo_hist_window_norm.argtypes = [vp, i64, i32, i32, i32, vp, vp]
        L.eqo_quantize_uniform.argtypes = [vp, i64, dbl, dbl, i32, i32, vp, vp, vp]
        L.eqo_pack_table4.argtypes = [vp, i64, i64, i32, vp, vp, vp]
        L.eqo_packed_row_stride.argtypes = [i64, i32]
        L.eqo_packed_row_stride.restype = i64
        L.eqo_quantize_pack_table.argtypes = [vp, i64, i64, i64, i32, i32, dbl, i32, vp, vp, vp,
                                              vp, vp, vp, i32]
        L.eqo_max_threads.restype = i32
        L.eqo_clip_range_sym.argtypes = [vp, i64, vp, vp]
        L.eqo_clip_range_aciq.argtypes = [vp, i64, vp, vp, vp]
        L.eqo_clip_range_gss.argtypes = [vp, i64, i32, vp, vp, vp, vp]
        L.eqo_sls4.argtypes = [vp, i64, i64, i32, vp, i64, vp, i64, vp, vp]
        L.eqo_quantize_pack_table_gaps.argtypes = [vp, i64, i64, i64, i32, i32, dbl, i32, vp, vp,
                                                   vp, vp, vp, vp, vp, vp, i32]
        L.eqo_np_extremum.argtypes = [vp, i64, i32]
        L.eqo_greedy_trace.argtypes = [vp, i64, i32, dbl, i32, vp, vp, vp, vp, vp, vp]
        L.eqo_np_extremum.restype = dbl
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32)


def max_threads() -> int:
    return int(lib().eqo_max_threads())


def np_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().eqo_np_sum(_p(a), a.size))


def np_extremum(x, is_max: bool) -> float:
    """np.min / np.max of a float32 row promoted to float64, numpy's zero-sign choice
    included (eq4_oracle.c np_reduce_ext)."""
    x = _f32(x)
    return float(lib().eqo_np_extremum(_p(x), x.size, int(bool(is_max))))


def quant_mse(x, xmin: float, xmax: float, nbits: int = 4) -> float:
    """table.py:81-103 (bit-exact)."""
    x = _f32(x)
    scratch = np.empty(max(1, x.size), np.float64)
    out = np.zeros(1, np.float64)
    rc = lib().eqo_quant_mse(_p(x), x.size, float(xmin), float(xmax), nbits, _p(scratch), _p(out))
    if rc:
        raise OracleError(rc)
    return float(out[0])


@dataclass
class GreedyResult:
    xmin: float
    xmax: float
    iters: int       # while-loop iterations; -1 = constant row (no loss evaluated)
    best_i: int      # returned xmin = x0 + best_i * step
    best_j: int      # returned xmax = x1 - best_j * step

    @property
    def loss_evals(self) -> int:
        return 0 if self.iters < 0 else 1 + 2 * self.iters


def clip_range_greedy(x, nbits: int = 4, b: int = 200, r: float = 0.16) -> GreedyResult:
    """clipping.py:142-193 (bit-exact)."""
    x = _f32(x)
    lo, hi = np.zeros(1), np.zeros(1)
    it, bi, bj = np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32)
    scratch = np.empty(max(16, x.size), np.float64)
    rc = lib().eqo_clip_range_greedy(_p(x), x.size, nbits, b, float(r), _p(lo), _p(hi), _p(it),
                                     _p(bi), _p(bj), _p(scratch))
    if rc:
        raise OracleError(rc)
    return GreedyResult(float(lo[0]), float(hi[0]), int(it[0]), int(bi[0]), int(bj[0]))


def build_histogram(x, b: int):
    """histclip.py:52-67 -> (lo, hi, counts int64)."""
    x = _f32(x)
    lo, hi = np.zeros(1), np.zeros(1)
    counts = np.zeros(b, np.int64)
    rc = lib().eqo_build_histogram(_p(x), x.size, b, _p(lo), _p(hi), _p(counts))
    if rc:
        raise OracleError(rc)
    return float(lo[0]), float(hi[0]), counts


@dataclass
class HistResult:
    xmin: float
    xmax: float
    start_bin: int
    nbins_selected: int
    norm: float
    candidate_evals: int
    bin_visits: int


def hist_brute_search(x, b: int = 200) -> HistResult:
    """histclip.py:136-174 (window selection pinned to the reference)."""
    x = _f32(x)
    lo, hi, norm = np.zeros(1), np.zeros(1), np.zeros(1)
    st, ns = np.zeros(1, np.int32), np.zeros(1, np.int32)
    ce, bv = np.zeros(1, np.int64), np.zeros(1, np.int64)
    scratch = np.empty(max(16, 5 * b), np.float64)
    rc = lib().eqo_hist_brute(_p(x), x.size, b, _p(lo), _p(hi), _p(st), _p(ns), _p(norm), _p(ce),
                              _p(bv), _p(scratch))
    if rc:
        raise OracleError(rc)
    return HistResult(float(lo[0]), float(hi[0]), int(st[0]), int(ns[0]), float(norm[0]),
                      int(ce[0]), int(bv[0]))


def hist_apprx_search(x, b: int = 200) -> HistResult:
    """histclip.py:181-217."""
    x = _f32(x)
    lo, hi, norm = np.zeros(1), np.zeros(1), np.zeros(1)
    st, ns = np.zeros(1, np.int32), np.zeros(1, np.int32)
    ce, bv = np.zeros(1, np.int64), np.zeros(1, np.int64)
    scratch = np.empty(max(16, 5 * b), np.float64)
    rc = lib().eqo_hist_apprx(_p(x), x.size, b, _p(lo), _p(hi), _p(st), _p(ns), _p(norm), _p(ce),
                              _p(bv), _p(scratch))
    if rc:
        raise OracleError(rc)
    return HistResult(float(lo[0]), float(hi[0]), int(st[0]), int(ns[0]), float(norm[0]),
                      int(ce[0]), int(bv[0]))


def hist_apprx_gap(x, b: int = 200):
    """(HistResult without counters, min relative |nl - nr| gap over the walk's decisions)."""
    x = _f32(x)
    lo, hi, norm, gap = np.zeros(1), np.zeros(1), np.zeros(1), np.zeros(1)
    st, ns = np.zeros(1, np.int32), np.zeros(1, np.int32)
    scratch = np.empty(max(16, 5 * b), np.float64)
    rc = lib().eqo_hist_apprx_gap(_p(x), x.size, b, _p(lo), _p(hi), _p(st), _p(ns), _p(norm),
                                  _p(scratch), _p(gap))
    if rc:
        raise OracleError(rc)
    return HistResult(float(lo[0]), float(hi[0]), int(st[0]), int(ns[0]), float(norm[0]), 0, 0), float(gap[0])


def hist_window_norm(x, b: int, start: int, n: int) -> float:
    """Norm of one (start, n) window as histclip.py:152-161 computes it (test helper)."""
    x = _f32(x)
    out = np.zeros(1)
    scratch = np.empty(max(16, 5 * b), np.float64)
    rc = lib().eqo_hist_window_norm(_p(x), x.size, b, start, n, _p(out), _p(scratch))
    if rc:
        raise OracleError(rc)
    return float(out[0])


def quantize_uniform(x, xmin: float, xmax: float, nbits: int = 4, aux: str = "fp32"):
    """uniform.py:60-80 -> (codes uint8, scale, bias) with scale/bias at the aux dtype."""
    x = _f32(x)
    codes = np.zeros(x.size, np.uint8)
    dt = np.float16 if aux == "fp16" else np.float32
    s, bb = np.zeros(1, dt), np.zeros(1, dt)
    rc = lib().eqo_quantize_uniform(_p(x), x.size, float(xmin), float(xmax), nbits, AUX[aux],
                                    _p(codes), _p(s), _p(bb))
    if rc:
        raise OracleError(rc)
    return codes, s[0], bb[0]


def packed_row_stride(d: int, aux: str) -> int:
    return int(lib().eqo_packed_row_stride(d, AUX[aux]))


def pack_table4(codes: np.ndarray, scales: np.ndarray, biases: np.ndarray, aux: str) -> np.ndarray:
    """packed.py:68-83 -> flat uint8 buffer."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n, d = codes.shape
    dt = np.float16 if aux == "fp16" else np.float32
    scales = np.ascontiguousarray(scales, dtype=dt)
    biases = np.ascontiguousarray(biases, dtype=dt)
    out = np.zeros(n * packed_row_stride(d, aux), np.uint8)
    lib().eqo_pack_table4(_p(codes), n, d, AUX[aux], _p(scales), _p(biases), _p(out))
    return out


@dataclass
class TableResult:
    packed: np.ndarray     # rows * stride bytes (packed.py layout)
    xmin: np.ndarray       # f64 per row
    xmax: np.ndarray
    info0: np.ndarray      # greedy: iterations (-1 constant); hist-brute: start_bin; gss: evals
    info1: np.ndarray      # greedy: best_i; hist-brute: nbins_selected
    norm: np.ndarray       # hist-brute window norm


def quantize_pack_table(x, method: str, b: int = 200, r: float = 0.16, aux: str = "fp16",
                        nthreads: int = 0) -> TableResult:
    """pack_table4(quantize_table(EmbeddingTable(x), method, 4, aux, b, r)) on host threads."""
    x = _f32(x)
    if x.ndim != 2:
        raise ValueError("expected a 2-D array")
    rows, d = x.shape
    packed = np.zeros(rows * packed_row_stride(d, aux), np.uint8)
    lo, hi, nv = np.zeros(rows), np.zeros(rows), np.zeros(rows)
    i0, i1 = np.zeros(rows, np.int32), np.zeros(rows, np.int32)
    rc = lib().eqo_quantize_pack_table(_p(x), rows, d, d, METHODS[method], b, float(r), AUX[aux],
                                       _p(packed), _p(lo), _p(hi), _p(i0), _p(i1), _p(nv),
                                       int(nthreads))
    if rc:
        raise OracleError(rc)
    return TableResult(packed, lo, hi, i0, i1, nv)


def greedy_trace(x, b: int = 200, r: float = 0.16, cap: int = 100000):
    """The reference walk of clip_range_greedy, step by step: (nl, nr, loss_l, loss_r) arrays
    with one entry per loop iteration (clipping.py:180-192)."""
    x = _f32(x)
    cap = min(cap, 2 * b + 2)
    nl, nr = np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    ll, lr = np.zeros(cap), np.zeros(cap)
    it = np.zeros(1, np.int32)
    scratch = np.empty(max(16, x.size), np.float64)
    rc = lib().eqo_greedy_trace(_p(x), x.size, b, float(r), cap, _p(it), _p(nl), _p(nr), _p(ll),
                                _p(lr), _p(scratch))
    if rc:
        raise OracleError(rc)
    n = int(it[0])
    return nl[:n], nr[:n], ll[:n], lr[:n]


def quantize_pack_table_gaps(x, b: int = 200, r: float = 0.16, aux: str = "fp16", nthreads: int = 0):
    """GREEDY table driver plus, per row, the smallest relative gap of the reference's two
    competing losses (clipping.py:185) and of candidate vs best (clipping.py:187,191) over
    the walk.  Returns (TableResult, gap_lr, gap_best)."""
    x = _f32(x)
    rows, d = x.shape
    packed = np.zeros(rows * packed_row_stride(d, aux), np.uint8)
    lo, hi, nv = np.zeros(rows), np.zeros(rows), np.zeros(rows)
    i0, i1 = np.zeros(rows, np.int32), np.zeros(rows, np.int32)
    g1, g2 = np.full(rows, np.inf), np.full(rows, np.inf)
    rc = lib().eqo_quantize_pack_table_gaps(_p(x), rows, d, d, METHODS["greedy"], b, float(r),
                                            AUX[aux], _p(packed), _p(lo), _p(hi), _p(i0), _p(i1),
                                            _p(nv), _p(g1), _p(g2), int(nthreads))
    if rc:
        raise OracleError(rc)
    return TableResult(packed, lo, hi, i0, i1, nv), g1, g2


def sparse_lengths_sum4(packed, rows: int, d: int, aux: str, indices, lengths):
    """packed.py:202-221 sparse_lengths_sum_ref over a PackedTable4 buffer.

    Returns (out float32 [batch x d], error code, bad position): error 0 = ok,
    9/10 = PooledQuery validation (packed.py:131-140), 11 = index out of range
    at `bad position` (packed.py:147-152)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    idx = np.ascontiguousarray(indices, dtype=np.int64).ravel()
    ln = np.ascontiguousarray(lengths, dtype=np.int64).ravel()
    out = np.zeros((ln.size, d), np.float32)
    bad = np.full(1, -1, np.int64)
    rc = lib().eqo_sls4(_p(packed), rows, d, AUX[aux], _p(idx), idx.size, _p(ln), ln.size,
                        _p(out), _p(bad))
    return out, int(rc), int(bad[0])


def clip_range_rowwise(x, method: str):
    """clipping.py sym / aciq (laplacian) / gss (tol 1e-4) for one row -> (lo, hi, evals)."""
    x = _f32(x)
    lo, hi = np.zeros(1), np.zeros(1)
    ev = np.zeros(1, np.int32)
    scratch = np.empty(max(16, x.size), np.float64)
    L = lib()
    if method == "sym":
        rc = L.eqo_clip_range_sym(_p(x), x.size, _p(lo), _p(hi))
    elif method == "aciq":
        rc = L.eqo_clip_range_aciq(_p(x), x.size, _p(scratch), _p(lo), _p(hi))
    elif method == "gss":
        rc = L.eqo_clip_range_gss(_p(x), x.size, 4, _p(scratch), _p(lo), _p(hi), _p(ev))
    else:
        raise ValueError(method)
    if rc:
        raise OracleError(rc)
    return float(lo[0]), float(hi[0]), int(ev[0])


def kmeans_table(x, aux: str = "fp32", nthreads: int = 0):
    """codebook.py:164-172 quantize_table_kmeans -> (codebooks (N,16) aux dtype, indices (N,d) u8,
    Lloyd rounds per row; -1 = the <= 16 distinct values shortcut)."""
    x = _f32(x)
    rows, d = x.shape
    dt = np.float16 if aux == "fp16" else np.float32
    books = np.zeros((rows, 16), dt)
    idx = np.zeros((rows, d), np.uint8)
    it = np.zeros(rows, np.int32)
    rc = lib().eqo_kmeans_table(_p(x), rows, d, d, AUX[aux], _p(books), _p(idx), _p(it), int(nthreads))
    if rc:
        raise OracleError(rc)
    return books, idx, it
