"""The reference's standalone codec, histogram and row-unpack entry points (B200 path).

Mirrors, with the same names, argument meaning, defaults and ValueError texts:
  - UniformRowQuant, quantize_uniform, dequantize_uniform   uniform.py:38-91
  - quantize_table_uniform                                  uniform.py:142-167
  - Histogram, build_histogram, bin_l2_norm                 histclip.py:34-82
  - unpack_row_codes, unpack_row                            packed.py:102-121
Every value is computed by libeq4.so on the GPU (eq4_quantize_rows,
eq4_dequantize_rows, eq4_build_histogram, eq4_bin_l2_norm, eq4_unpack); inputs
are promoted to float64 like the reference's np.asarray(x, dtype=np.float64)
(float32 EmbeddingTable rows stay float32 on the device -- the same values).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .api import (AUX_PRECISIONS, ClipRange, EmbeddingTable, PackedTable4, UniformQuantTable,
                  _AUX_NP, _check_aux, _is_cuda, _rows_on_device, _stream_handle, _vp, pack_table4)

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def aux_dtype(aux_precision: str):
    """uniform.py:25-29."""
    try:
        return _AUX_NP[aux_precision]
    except KeyError:
        raise ValueError(f"aux_precision must be one of {AUX_PRECISIONS}, got {aux_precision!r}") from None


# ---------------------------------------------------------------------------
# uniform.py
# ---------------------------------------------------------------------------
@dataclass
class UniformRowQuant:
    """One quantized row: codes plus its stored scale/bias (uniform.py:38-57)."""

    codes: np.ndarray
    scale: np.floating
    bias: np.floating
    nbits: int

    def __post_init__(self):
        self.codes = np.asarray(self.codes, dtype=np.uint8)
        if self.nbits not in (4, 8):
            raise ValueError(f"nbits must be 4 or 8, got {self.nbits}")
        if self.codes.size and int(self.codes.max()) > (1 << self.nbits) - 1:
            raise ValueError(f"codes exceed {self.nbits}-bit range")


def _quantize_rows(t, is_f64, lo, hi, nbits, aux_precision):
    """Device codes/scales/biases of rows t against float64 ranges lo/hi (length 1 or rows)."""
    rows, d = int(t.shape[0]), int(t.shape[1])
    dev = t.device
    lo_t = torch.as_tensor(np.ascontiguousarray(lo, dtype=np.float64)).to(dev)
    hi_t = torch.as_tensor(np.ascontiguousarray(hi, dtype=np.float64)).to(dev)
    codes = torch.empty((rows, d), dtype=torch.uint8, device=dev)
    adt = torch.float16 if aux_precision == "fp16" else torch.float32
    sc = torch.empty(rows, dtype=adt, device=dev)
    bi = torch.empty(rows, dtype=adt, device=dev)
    _lib.check(_lib.load().eq4_quantize_rows(
        _vp(t), int(is_f64), rows, d, d, _vp(lo_t), _vp(hi_t), 0 if lo_t.numel() == 1 else 1, nbits,
        _lib.AUX[aux_precision], _vp(codes), _vp(sc), _vp(bi), _stream_handle()))
    return codes, sc, bi


def quantize_uniform(x, clip_range: ClipRange, nbits: int, aux_precision: str = "fp32") -> UniformRowQuant:
    """uniform.py:60-80: codes of x against clip_range (float64 scale/bias, half-up rounding);
    only the stored scale/bias are rounded to the aux width.  Degenerate range: scale 0,
    codes 0."""
    if nbits not in (4, 8):
        raise ValueError(f"nbits must be 4 or 8, got {nbits}")
    aux_dtype(aux_precision)
    shape = tuple(x.shape) if _is_cuda(x) else np.shape(x)
    flat = x.reshape(-1) if _is_cuda(x) else np.asarray(x).reshape(-1)
    n = int(flat.numel() if _is_cuda(x) else flat.size)
    t, f64 = _rows_on_device(flat if n else np.zeros(1))   # an empty x still gets its scale/bias
    codes, sc, bi = _quantize_rows(t, f64, [clip_range.xmin], [clip_range.xmax], nbits, aux_precision)
    c = codes.cpu().numpy()[0][:n].reshape(shape)
    return UniformRowQuant(c, sc.cpu().numpy()[0], bi.cpu().numpy()[0], nbits)


def dequantize_uniform(q: UniformRowQuant) -> np.ndarray:
    """uniform.py:83-91: float32(scale) * code + float32(bias), in float32 (GPU)."""
    shape = np.shape(q.codes)
    codes = np.ascontiguousarray(np.asarray(q.codes, dtype=np.uint8).reshape(1, -1))
    if codes.size == 0:
        return np.zeros(shape, np.float32)
    aux = "fp16" if np.asarray(q.scale).dtype == np.float16 else "fp32"
    dt = _AUX_NP[aux]
    dev_codes = torch.from_numpy(codes).cuda()
    sc = torch.from_numpy(np.array([q.scale], dtype=dt).view(np.uint8)).cuda()
    bi = torch.from_numpy(np.array([q.bias], dtype=dt).view(np.uint8)).cuda()
    out = torch.empty(codes.shape, dtype=torch.float32, device=dev_codes.device)
    _lib.check(_lib.load().eq4_dequantize_rows(_vp(dev_codes), 1, codes.shape[1], _vp(sc), _vp(bi),
                                               _lib.AUX[aux], _vp(out), _stream_handle()))
    return out.cpu().numpy()[0].reshape(shape)


def quantize_table_uniform(table, ranges, nbits: int, aux_precision: str = "fp32",
                           scheme: str = "asym") -> UniformQuantTable:
    """uniform.py:142-167: every row against its ClipRange (or one ClipRange for all rows);
    codes, scales and biases of the whole table come from one launch (eq4_quantize_rows)."""
    _check_aux(aux_precision)
    if not isinstance(table, EmbeddingTable):
        table = EmbeddingTable(table)
    if isinstance(ranges, ClipRange):
        ranges = [ranges] * table.rows
    if len(ranges) != table.rows:
        raise ValueError(f"expected {table.rows} ranges, got {len(ranges)}")
    if nbits not in (4, 8):
        raise ValueError(f"nbits must be 4 or 8, got {nbits}")
    lo = np.array([r.xmin for r in ranges], dtype=np.float64)
    hi = np.array([r.xmax for r in ranges], dtype=np.float64)
    t, f64 = _rows_on_device(table)
    codes, sc, bi = _quantize_rows(t, f64, lo, hi, nbits, aux_precision)
    return UniformQuantTable(codes.cpu().numpy(), sc.cpu().numpy(), bi.cpu().numpy(), nbits,
                             aux_precision, scheme)


# ---------------------------------------------------------------------------
# histclip.py
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Histogram:
    """Counts over b equal bins spanning [lo, hi]; the last bin is closed (histclip.py:34-49)."""

    nbins: int
    lo: float
    hi: float
    counts: np.ndarray

    @property
    def bin_width(self) -> float:
        return (self.hi - self.lo) / self.nbins

    def centers(self) -> np.ndarray:
        w = self.bin_width
        return self.lo + w * (np.arange(self.nbins) + 0.5)


def build_histogram(x, b: int) -> Histogram:
    """histclip.py:52-67, computed on the GPU (np.min / np.max incl. numpy's zero choice,
    float64 bin index, int64 counts)."""
    if b < 1:
        raise ValueError(f"b must be >= 1, got {b}")
    if not _is_cuda(x) and np.asarray(x).size == 0:
        raise ValueError("input vector is empty")
    t, f64 = _rows_on_device(np.asarray(x).reshape(-1) if not _is_cuda(x) else x.reshape(-1))
    if t.numel() == 0:
        raise ValueError("input vector is empty")
    d = int(t.shape[1])
    dev = t.device
    lo = torch.empty(1, dtype=torch.float64, device=dev)
    hi = torch.empty(1, dtype=torch.float64, device=dev)
    counts = torch.empty(b, dtype=torch.int64, device=dev)
    _lib.check(_lib.load().eq4_build_histogram(_vp(t), int(f64), 1, d, d, int(b), _vp(lo), _vp(hi),
                                               _vp(counts), _stream_handle()))
    return Histogram(int(b), float(lo.item()), float(hi.item()), counts.cpu().numpy())


def bin_l2_norm(delta_begin, delta_end, density):
    """histclip.py:70-82: density * (delta_end**3 - delta_begin**3) / 3.0 (scalars or
    arrays, numpy broadcasting), elementwise on the GPU."""
    db = np.asarray(delta_begin, dtype=np.float64)
    de = np.asarray(delta_end, dtype=np.float64)
    rho = np.asarray(density, dtype=np.float64)
    db, de, rho = np.broadcast_arrays(db, de, rho)
    shape = db.shape
    n = int(db.size)
    if n == 0:
        return np.zeros(shape, np.float64)
    dev_in = [torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).cuda() for a in (db, de, rho)]
    out = torch.empty(n, dtype=torch.float64, device=dev_in[0].device)
    _lib.check(_lib.load().eq4_bin_l2_norm(_vp(dev_in[0]), _vp(dev_in[1]), _vp(dev_in[2]), n, _vp(out),
                                           _stream_handle()))
    res = out.cpu().numpy().reshape(shape)
    if res.ndim == 0:
        return float(res)
    return res


# ---------------------------------------------------------------------------
# packed.py row unpacking
# ---------------------------------------------------------------------------
def unpack_row_codes(p: PackedTable4, i: int):
    """packed.py:102-115: (codes, scale, bias) of row i, scale/bias at the stored width
    (decoded on the GPU by eq4_unpack)."""
    if not 0 <= i < p.rows:
        raise IndexError(f"row index {i} out of range for {p.rows} rows")
    dev = p.to_device()
    stride = p.row_stride
    row = dev[i * stride:(i + 1) * stride]
    codes = torch.empty((1, p.dim), dtype=torch.uint8, device=dev.device)
    dt = torch.float16 if p.aux_precision == "fp16" else torch.float32
    sc = torch.empty(1, dtype=dt, device=dev.device)
    bi = torch.empty(1, dtype=dt, device=dev.device)
    _lib.check(_lib.load().eq4_unpack(_vp(row), 1, p.dim, _lib.AUX[p.aux_precision], _vp(codes), _vp(sc),
                                      _vp(bi), _stream_handle()))
    return codes.cpu().numpy()[0], sc.cpu().numpy()[0], bi.cpu().numpy()[0]


def unpack_row(p: PackedTable4, i: int) -> np.ndarray:
    """packed.py:118-121: dequantized row i, float32 scale * code + bias (GPU)."""
    codes, scale, bias = unpack_row_codes(p, i)
    return dequantize_uniform(UniformRowQuant(codes, scale, bias, 4))


__all__ = ["Histogram", "UniformRowQuant", "bin_l2_norm", "build_histogram", "dequantize_uniform",
           "quantize_table_uniform", "quantize_uniform", "unpack_row", "unpack_row_codes", "aux_dtype",
           "pack_table4"]
