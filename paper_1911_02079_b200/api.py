"""Drop-in host API for the reference's quantize entry points (B200 path).

Mirrors the reference package `embquant` for the hot path:
  - EmbeddingTable, ClipRange           table.py:12-78
  - WorkCounters                        clipping.py:30-41
  - quantize_table, row_clip_range      methods.py:43-89
  - clip_range_asym / clip_range_greedy clipping.py:58-61, 142-193
  - hist_brute_search / HistWindow / clip_range_hist_brute   histclip.py:126-178
  - UniformQuantTable                   uniform.py:94-139
  - PackedTable4, pack_table4, packed_row_stride   packed.py:32-83
  - quant_mse                           table.py:81-103
Same names, argument meaning, defaults and ValueError texts.  Every result is
computed by libeq4.so on the GPU (device tables stay in HBM; host tables go
through the pipelined host entry point); methods outside the hot path raise.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

UNIFORM_METHODS = ("sym", "asym", "table", "gss", "aciq", "greedy", "hist-apprx", "hist-brute")
CODEBOOK_METHODS = ("kmeans", "kmeans-cls")
ALL_METHODS = UNIFORM_METHODS + CODEBOOK_METHODS            # methods.py:38-40
GPU_METHODS = ("sym", "asym", "table", "gss", "aciq", "greedy", "hist-apprx", "hist-brute")
AUX_PRECISIONS = ("fp32", "fp16")                            # uniform.py:19
_AUX_NP = {"fp32": np.float32, "fp16": np.float16}


def _vp(x) -> ctypes.c_void_p | None:
    if x is None:
        return None
    if torch is not None and isinstance(x, torch.Tensor):
        return ctypes.c_void_p(x.data_ptr())
    return x.ctypes.data_as(ctypes.c_void_p)


def _stream_handle(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _is_cuda(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _rows_on_device(x):
    """(device tensor rows x d, is_f64) of an array-like promoted like np.asarray(x, float64).

    float32 inputs (EmbeddingTable rows, float32 arrays/tensors) stay float32 -- promoting
    them to float64 is exact; anything else becomes a float64 tensor."""
    if isinstance(x, EmbeddingTable):
        x = x.device_values if x.on_device else x.values
    if _is_cuda(x):
        t = x if x.dtype in (torch.float32, torch.float64) else x.double()
    else:
        a = np.asarray(x)
        if a.dtype != np.float32:
            a = np.asarray(x, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    if t.dim() == 1:
        t = t.reshape(1, -1)
    t = t.contiguous()
    return t, t.dtype == torch.float64


# ---------------------------------------------------------------------------
# containers (table.py)
# ---------------------------------------------------------------------------
class EmbeddingTable:
    """Dense N x d float32 table (table.py:12-60).

    Accepts anything numpy accepts (host) or a CUDA ``torch.Tensor`` (kept in
    HBM).  Values must be finite: a host table is checked here, as the
    reference does (table.py:28-29); a device table is checked by the kernels
    themselves while they read it (their status word), so the same ValueError
    surfaces from the first quantize call without an extra pass over HBM or a
    host synchronisation at construction.
    """

    __slots__ = ("_values", "_device")

    def __init__(self, values):
        if _is_cuda(values):
            t = values
            if t.dim() != 2:
                raise ValueError(f"expected a 2-D array, got shape {tuple(t.shape)}")
            if t.shape[0] < 1 or t.shape[1] < 1:
                raise ValueError(f"table must be at least 1x1, got shape {tuple(t.shape)}")
            if t.dtype != torch.float32 or not t.is_contiguous():
                t = t.to(torch.float32).contiguous()
            self._device = t
            self._values = None
            return
        if torch is not None and isinstance(values, torch.Tensor):
            values = values.numpy()
        arr = np.ascontiguousarray(values, dtype=np.float32)
        if arr.ndim != 2:
            raise ValueError(f"expected a 2-D array, got shape {arr.shape}")
        if arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ValueError(f"table must be at least 1x1, got shape {arr.shape}")
        if not np.all(np.isfinite(arr)):
            raise ValueError("table contains non-finite values (NaN/Inf)")
        arr.flags.writeable = False
        self._values = arr
        self._device = None

    @property
    def on_device(self) -> bool:
        return self._device is not None

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            v = self._device.cpu().numpy()
            v.flags.writeable = False
            return v
        return self._values

    @property
    def device_values(self):
        return self._device

    @property
    def rows(self) -> int:
        return int((self._device if self._device is not None else self._values).shape[0])

    @property
    def dim(self) -> int:
        return int((self._device if self._device is not None else self._values).shape[1])

    def row(self, i: int) -> np.ndarray:
        if not 0 <= i < self.rows:
            raise IndexError(f"row index {i} out of range for table with {self.rows} rows")
        return self.values[i]

    def __repr__(self):
        where = "cuda" if self.on_device else "host"
        return f"EmbeddingTable(rows={self.rows}, dim={self.dim}, {where})"


@dataclass(frozen=True)
class ClipRange:
    """Clamp interval [xmin, xmax] (table.py:63-78)."""

    xmin: float
    xmax: float

    def __post_init__(self):
        if not (np.isfinite(self.xmin) and np.isfinite(self.xmax)):
            raise ValueError(f"clip range must be finite, got ({self.xmin}, {self.xmax})")
        if self.xmin > self.xmax:
            raise ValueError(f"xmin {self.xmin} exceeds xmax {self.xmax}")

    @property
    def width(self) -> float:
        return self.xmax - self.xmin


@dataclass
class WorkCounters:
    """Instrumented work totals (clipping.py:30-41)."""

    loss_evals: int = 0
    candidate_evals: int = 0
    bin_visits: int = 0

    def merge(self, other: "WorkCounters") -> None:
        self.loss_evals += other.loss_evals
        self.candidate_evals += other.candidate_evals
        self.bin_visits += other.bin_visits


@dataclass(frozen=True)
class HistWindow:
    """histclip.py:126-133."""

    clip_range: ClipRange
    start_bin: int
    nbins_selected: int
    norm: float


# ---------------------------------------------------------------------------
# packed format (packed.py)
# ---------------------------------------------------------------------------
def packed_row_stride(dim: int, aux_precision: str) -> int:
    """packed.py:32-33."""
    _check_aux(aux_precision)
    return (dim + 1) // 2 + 2 * (2 if aux_precision == "fp16" else 4)


class PackedTable4:
    """N fused rows of packed nibbles + scale + bias (packed.py:36-65).

    ``buffer`` is the host uint8 view (materialised from HBM on first access
    when the table was quantized on the device); ``device_buffer`` is the
    CUDA uint8 tensor when one exists.
    """

    def __init__(self, rows: int, dim: int, aux_precision: str, buffer=None, device_buffer=None):
        self.rows = int(rows)
        self.dim = int(dim)
        self.aux_precision = aux_precision
        self._buffer = None
        self.device_buffer = device_buffer
        expected = self.rows * self.row_stride
        if buffer is not None:
            buf = np.asarray(buffer, dtype=np.uint8).reshape(-1)
            if buf.size != expected:
                raise ValueError(f"buffer has {buf.size} bytes, expected {expected}")
            self._buffer = buf
        elif device_buffer is None:
            raise ValueError("PackedTable4 needs a host or a device buffer")
        elif device_buffer.numel() != expected:
            raise ValueError(f"buffer has {device_buffer.numel()} bytes, expected {expected}")

    @property
    def row_stride(self) -> int:
        return packed_row_stride(self.dim, self.aux_precision)

    @property
    def buffer(self) -> np.ndarray:
        if self._buffer is None:
            self._buffer = self.device_buffer.cpu().numpy().reshape(-1)
        return self._buffer

    @property
    def nbytes(self) -> int:
        return self.rows * self.row_stride

    def tobytes(self) -> bytes:
        return self.buffer.tobytes()

    def to_device(self):
        if self.device_buffer is None:
            self.device_buffer = torch.from_numpy(np.ascontiguousarray(self._buffer)).cuda()
        return self.device_buffer

    def unpack(self):
        """(codes (N,d) uint8, scales, biases) at the aux dtype, decoded on the GPU."""
        dev = self.to_device()
        codes = torch.empty((self.rows, self.dim), dtype=torch.uint8, device=dev.device)
        dt = torch.float16 if self.aux_precision == "fp16" else torch.float32
        sc = torch.empty(self.rows, dtype=dt, device=dev.device)
        bi = torch.empty(self.rows, dtype=dt, device=dev.device)
        _lib.check(_lib.load().eq4_unpack(_vp(dev), self.rows, self.dim, _lib.AUX[self.aux_precision],
                                          _vp(codes), _vp(sc), _vp(bi), _stream_handle()))
        return codes, sc, bi

    def dequantize(self) -> np.ndarray:
        codes, sc, bi = self.unpack()
        out = sc.float()[:, None] * codes.float() + bi.float()[:, None]
        return out.cpu().numpy()


class UniformQuantTable:
    """Per-row codes + scale/bias (uniform.py:94-139).

    Built either like the reference (codes, scales, biases arrays) or from a
    GPU-packed table (``UniformQuantTable.from_packed``); codes/scales/biases
    of a packed table are decoded on the GPU on first access.
    """

    def __init__(self, codes=None, scales=None, biases=None, nbits: int = 4,
                 aux_precision: str = "fp32", scheme: str = "asym", *, packed: PackedTable4 = None):
        _check_aux(aux_precision)
        self.nbits = nbits
        self.aux_precision = aux_precision
        self.scheme = scheme
        self._packed = packed
        if packed is None:
            dt = _AUX_NP[aux_precision]
            self._codes = np.asarray(codes, dtype=np.uint8)
            self._scales = np.asarray(scales, dtype=dt)
            self._biases = np.asarray(biases, dtype=dt)
            if self._codes.ndim != 2:
                raise ValueError("codes must be a 2-D (rows, dim) array")
            n = self._codes.shape[0]
            if self._scales.shape != (n,) or self._biases.shape != (n,):
                raise ValueError("scales/biases must be length-N vectors")
        else:
            self._codes = self._scales = self._biases = None

    @classmethod
    def from_packed(cls, packed: PackedTable4, scheme: str) -> "UniformQuantTable":
        return cls(nbits=4, aux_precision=packed.aux_precision, scheme=scheme, packed=packed)

    def _decode(self):
        if self._codes is None:
            c, s, b = self._packed.unpack()
            self._codes, self._scales, self._biases = c.cpu().numpy(), s.cpu().numpy(), b.cpu().numpy()

    @property
    def codes(self) -> np.ndarray:
        self._decode()
        return self._codes

    @property
    def scales(self) -> np.ndarray:
        self._decode()
        return self._scales

    @property
    def biases(self) -> np.ndarray:
        self._decode()
        return self._biases

    @property
    def rows(self) -> int:
        return self._packed.rows if self._packed is not None else self._codes.shape[0]

    @property
    def dim(self) -> int:
        return self._packed.dim if self._packed is not None else self._codes.shape[1]

    @property
    def packed(self) -> PackedTable4 | None:
        return self._packed

    def dequantize(self) -> np.ndarray:
        scales = self.scales.astype(np.float32)[:, None]
        biases = self.biases.astype(np.float32)[:, None]
        return scales * self.codes.astype(np.float32) + biases


def pack_table4(q: UniformQuantTable) -> PackedTable4:
    """packed.py:68-83.  A GPU-quantized table is already packed (zero copy)."""
    if q.nbits != 4:
        raise ValueError(f"packing requires 4-bit codes, got nbits={q.nbits}")
    if q.packed is not None:
        return q.packed
    n, d = q.rows, q.dim
    codes = torch.from_numpy(np.ascontiguousarray(q.codes)).cuda()
    dt = _AUX_NP[q.aux_precision]
    sc = torch.from_numpy(np.ascontiguousarray(q.scales, dtype=dt).view(np.uint8)).cuda()
    bi = torch.from_numpy(np.ascontiguousarray(q.biases, dtype=dt).view(np.uint8)).cuda()
    out = torch.empty(n * packed_row_stride(d, q.aux_precision), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.load().eq4_pack(_vp(codes), n, d, _lib.AUX[q.aux_precision], _vp(sc), _vp(bi),
                                    _vp(out), _stream_handle()))
    return PackedTable4(n, d, q.aux_precision, device_buffer=out)


# ---------------------------------------------------------------------------
# the fused hot path
# ---------------------------------------------------------------------------
def _check_aux(aux):
    if aux not in AUX_PRECISIONS:
        raise ValueError(f"aux_precision must be one of {AUX_PRECISIONS}, got {aux!r}")


def _check_method_params(method: str, b: int, r: float) -> None:
    if method == "greedy":
        if b < 1:
            raise ValueError(f"b must be >= 1, got {b}")            # clipping.py:158-159
        if not 0.0 < r <= 1.0:
            raise ValueError(f"r must be in (0, 1], got {r}")       # clipping.py:160-161
    elif method in ("hist-brute", "hist-apprx") and b < 1:
        raise ValueError(f"b must be >= 1, got {b}")                # histclip.py:54-55


@dataclass
class RowResults:
    """Per-row outputs of one fused launch (device or host arrays)."""

    xmin: object = None
    xmax: object = None
    info0: object = None
    info1: object = None
    norm: object = None


def quantize_pack_table4(table, method: str, aux_precision: str = "fp16", b: int = 200,
                         r: float = 0.16, *, out=None, rows_out: RowResults | None = None,
                         with_rows: bool = False, status=None, stream=None, check: bool = True,
                         param: float = 0.0):
    """Fused ``pack_table4(quantize_table(table, method, 4, aux, b, r))`` on the GPU.

    ``table``: EmbeddingTable, CUDA float32 tensor (device path, stream
    ordered) or host array (pipelined host path).  Returns
    ``(PackedTable4, RowResults | None)``.  With ``check=False`` on the device
    path nothing synchronises; the caller inspects ``status`` itself (the C
    entry point clears it on the stream first).  ``stream`` (a torch CUDA
    stream, default the current one) orders the launch; the output buffers
    are allocated on it and the status read waits for it.  ``param``: ACIQ's
    clipping constant / GSS's tol (0 = the reference defaults 5.03 / 1e-4;
    device tables only).
    """
    if method not in GPU_METHODS:
        raise ValueError(f"{method!r} is not on the B200 hot path; supported: {GPU_METHODS}")
    _check_aux(aux_precision)
    _check_method_params(method, b, r)
    L = _lib.load()
    if isinstance(table, EmbeddingTable):
        src = table.device_values if table.on_device else table.values
    else:
        src = table
    if _is_cuda(src):
        if stream is not None and stream != torch.cuda.current_stream(src.device):
            with torch.cuda.stream(stream):
                return quantize_pack_table4(src, method, aux_precision, b, r, out=out, rows_out=rows_out,
                                            with_rows=with_rows, status=status, stream=None, check=check,
                                            param=param)
        x = src if (src.dtype == torch.float32 and src.stride(1) == 1) else src.float().contiguous()
        rows, d = int(x.shape[0]), int(x.shape[1])
        ld = int(x.stride(0))
        dev = x.device
        stride = packed_row_stride(d, aux_precision)
        if out is None:
            out = torch.empty(rows * stride, dtype=torch.uint8, device=dev)
        rr = rows_out
        if rr is None and with_rows:
            rr = RowResults(torch.empty(rows, dtype=torch.float64, device=dev),
                            torch.empty(rows, dtype=torch.float64, device=dev),
                            torch.empty(rows, dtype=torch.int32, device=dev),
                            torch.empty(rows, dtype=torch.int32, device=dev),
                            torch.empty(rows, dtype=torch.float64, device=dev))
        if status is None:
            status = torch.empty(1, dtype=torch.int32, device=dev)   # cleared by eq4_quantize_pack
        rc = L.eq4_quantize_pack_p(_vp(x), rows, d, ld, _lib.METHOD[method], int(b), float(r),
                                   float(param), _lib.AUX[aux_precision], _vp(out),
                                 _vp(rr.xmin) if rr else None, _vp(rr.xmax) if rr else None,
                                 _vp(rr.info0) if rr else None, _vp(rr.info1) if rr else None,
                                 _vp(rr.norm) if rr else None, _vp(status), _stream_handle(stream))
        _lib.check(rc)
        if check:
            st = int(status.item())
            if st:
                _raise_status(st, x, method, b, r, aux_precision)
        return PackedTable4(rows, d, aux_precision, device_buffer=out), rr
    if param:
        raise ValueError("param (ACIQ constant / GSS tol) is taken on the device path only")
    # host path: pinned/pageable host memory through the pipelined C entry point
    if torch is not None and isinstance(src, torch.Tensor):
        xh = src.float().contiguous().numpy()
    else:
        xh = np.ascontiguousarray(src, dtype=np.float32)
    if xh.ndim != 2:
        raise ValueError(f"expected a 2-D array, got shape {xh.shape}")
    rows, d = xh.shape
    stride = packed_row_stride(d, aux_precision)
    if out is None:
        out = np.empty(rows * stride, dtype=np.uint8)
    rr = rows_out
    if rr is None and with_rows:
        rr = RowResults(np.empty(rows), np.empty(rows), np.empty(rows, np.int32),
                        np.empty(rows, np.int32), np.empty(rows))
    bad = np.full(1, -1, np.int64)
    badlh = np.zeros(2)
    rc = L.eq4_quantize_pack_host(_vp(xh), rows, d, d, _lib.METHOD[method], int(b), float(r),
                                  _lib.AUX[aux_precision], _vp(out),
                                  _vp(rr.xmin) if rr else None, _vp(rr.xmax) if rr else None,
                                  _vp(rr.info0) if rr else None, _vp(rr.info1) if rr else None,
                                  _vp(rr.norm) if rr else None, 0, _vp(bad), _vp(badlh))
    if rc == _lib.EQ4_ERANGE:
        raise ValueError(f"xmin {float(badlh[0])} exceeds xmax {float(badlh[1])}")
    _lib.check(rc)
    return PackedTable4(rows, d, aux_precision, buffer=out), rr


def _raise_status(st: int, x, method, b, r, aux):
    """Re-derive the reference's exception for a failed device launch."""
    if st & _lib.STATUS_NONFINITE:
        raise ValueError("table contains non-finite values (NaN/Inf)")
    if st & _lib.STATUS_RANGE:
        _, rr = quantize_pack_table4(x, method, aux, b, r, with_rows=True, check=False)
        i0 = rr.info0.cpu().numpy()
        first = int(np.nonzero(i0 == -2)[0][0])
        lo, hi = float(rr.xmin[first].item()), float(rr.xmax[first].item())
        raise ValueError(f"xmin {lo} exceeds xmax {hi}")
    raise _lib.Eq4Error(f"unknown status {st}")


def _apply_counters(counters: WorkCounters, method: str, b: int, rr: RowResults) -> None:
    if counters is None or method in ("asym", "sym", "aciq", "table"):
        return
    if method == "gss":                                             # clipping.py:87-89
        ev = np.asarray(rr.info0.cpu() if _is_cuda(rr.info0) else rr.info0).astype(np.int64)
        counters.loss_evals += int(ev.sum())
        return
    if method == "hist-apprx":                                      # histclip.py:113-115,193-210
        lo = np.asarray(rr.xmin.cpu() if _is_cuda(rr.xmin) else rr.xmin)
        hi = np.asarray(rr.xmax.cpu() if _is_cuda(rr.xmax) else rr.xmax)
        const = int(np.sum(lo == hi))
        full = lo.size - const
        counters.candidate_evals += full * (2 * b - 1) + const
        counters.bin_visits += full * (2 * b - 1) * b + const * b
        return
    if method == "greedy":                                          # clipping.py:174,183-184
        it = np.asarray(rr.info0.cpu() if _is_cuda(rr.info0) else rr.info0).astype(np.int64)
        counters.loss_evals += int(np.sum(np.where(it >= 0, 1 + 2 * it, 0)))
    else:                                                           # histclip.py:148-150,162-164
        lo = np.asarray(rr.xmin.cpu() if _is_cuda(rr.xmin) else rr.xmin)
        hi = np.asarray(rr.xmax.cpu() if _is_cuda(rr.xmax) else rr.xmax)
        const = int(np.sum(lo == hi))
        full = lo.size - const
        ncand = b * (b + 1) // 2
        counters.candidate_evals += full * ncand + const
        counters.bin_visits += full * ncand * b + const * b


def quantize_table(table, method: str, nbits: int = 4, aux_precision: str = "fp32", b: int = 200,
                   r: float = 0.16, k: int | None = None, seed: int = 0,
                   counters: WorkCounters | None = None) -> UniformQuantTable:
    """methods.py:63-89: every uniform method (GPU_METHODS) and row-wise kmeans at 4 bits."""
    if method not in ALL_METHODS:
        raise ValueError(f"unknown method {method!r}; expected one of {ALL_METHODS}")
    if method in CODEBOOK_METHODS and nbits != 4:
        raise ValueError(f"{method} is 4-bit only, got nbits={nbits}")
    if k is not None and method != "kmeans-cls":
        raise ValueError(f"k applies only to kmeans-cls, not {method}")
    if method == "kmeans":                                          # methods.py:76-77
        from .codebook import quantize_table_kmeans

        return quantize_table_kmeans(table, aux_precision)
    if method not in GPU_METHODS or nbits != 4:
        raise ValueError(f"{method!r} with nbits={nbits} is not on the B200 hot path "
                         f"(supported: {GPU_METHODS + ('kmeans',)} at nbits=4)")
    _check_aux(aux_precision)
    if not isinstance(table, EmbeddingTable):
        table = EmbeddingTable(table)
    packed, rr = quantize_pack_table4(table, method, aux_precision, b, r,
                                      with_rows=counters is not None)
    _apply_counters(counters, method, b, rr)
    return UniformQuantTable.from_packed(packed, scheme=method)


def _one_row(x):
    """The row as the reference sees it (np.asarray(x, float64), clipping.py:44-48): a float32
    (1, d) array/tensor when its values are float32 values (every EmbeddingTable row), else a
    float64 one."""
    if _is_cuda(x):
        x = x.reshape(1, -1)
        if x.numel() == 0:
            raise ValueError("input vector is empty")
        if x.dtype == torch.float32:
            return x
        x = x.double()
        return x.float() if bool((x.float().double() == x).all()) else x
    a = np.asarray(x)
    if a.size == 0:
        raise ValueError("input vector is empty")                  # clipping.py:44-48
    if a.dtype == np.float32:
        return a.reshape(1, -1)
    a = np.asarray(x, dtype=np.float64).reshape(1, -1)
    f = a.astype(np.float32)
    return f if np.array_equal(f.astype(np.float64), a, equal_nan=True) else a


def _row_search(method, x, b=200, r=0.16, param=0.0):
    row = _one_row(x)
    if not _is_cuda(row):
        row = torch.from_numpy(np.ascontiguousarray(row)).cuda()
    if row.dtype == torch.float64:
        # values that are not float32 values: the reference searches them in float64
        if method not in ("aciq", "gss"):
            raise ValueError(f"{method}: the B200 path takes float32 rows (every EmbeddingTable "
                             "row is one); this float64 row has values float32 cannot hold")
        dev = row.device
        n = int(row.shape[1])
        rr = RowResults(torch.empty(1, dtype=torch.float64, device=dev),
                        torch.empty(1, dtype=torch.float64, device=dev),
                        torch.empty(1, dtype=torch.int32, device=dev), None, None)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        _lib.check(_lib.load().eq4_row_range_f64(_vp(row), 1, n, n, _lib.METHOD[method], float(param),
                                                 _vp(rr.xmin), _vp(rr.xmax), _vp(rr.info0), _vp(st),
                                                 _stream_handle()))
        if int(st.item()) & _lib.STATUS_NONFINITE:
            raise ValueError("clip range must be finite")
        return rr
    _, rr = quantize_pack_table4(row, method, "fp32", b, r, with_rows=True, param=param)
    return rr


def clip_range_asym(x) -> ClipRange:
    """clipping.py:58-61."""
    rr = _row_search("asym", x)
    return ClipRange(float(rr.xmin[0].item()), float(rr.xmax[0].item()))


def clip_range_greedy(x, nbits: int = 4, b: int = 200, r: float = 0.16,
                      counters: WorkCounters | None = None) -> ClipRange:
    """clipping.py:142-193."""
    _check_method_params("greedy", b, r)
    if nbits != 4:
        raise ValueError(f"nbits={nbits} is not on the B200 hot path (4-bit only)")
    rr = _row_search("greedy", x, b, r)
    _apply_counters(counters, "greedy", b, rr)
    return ClipRange(float(rr.xmin[0].item()), float(rr.xmax[0].item()))


def hist_brute_search(x, b: int = 200, counters: WorkCounters | None = None) -> HistWindow:
    """histclip.py:136-174."""
    _check_method_params("hist-brute", b, 0.16)
    rr = _row_search("hist-brute", x, b)
    _apply_counters(counters, "hist-brute", b, rr)
    return HistWindow(ClipRange(float(rr.xmin[0].item()), float(rr.xmax[0].item())),
                      int(rr.info0[0].item()), int(rr.info1[0].item()), float(rr.norm[0].item()))


def hist_apprx_search(x, b: int = 200, counters: WorkCounters | None = None) -> HistWindow:
    """histclip.py:181-217."""
    _check_method_params("hist-apprx", b, 0.16)
    rr = _row_search("hist-apprx", x, b)
    _apply_counters(counters, "hist-apprx", b, rr)
    return HistWindow(ClipRange(float(rr.xmin[0].item()), float(rr.xmax[0].item())),
                      int(rr.info0[0].item()), int(rr.info1[0].item()), float(rr.norm[0].item()))


def clip_range_hist_apprx(x, b: int = 200, counters: WorkCounters | None = None) -> ClipRange:
    """histclip.py:220-221."""
    return hist_apprx_search(x, b, counters).clip_range


def clip_range_hist_brute(x, b: int = 200, counters: WorkCounters | None = None) -> ClipRange:
    """histclip.py:177-178."""
    return hist_brute_search(x, b, counters).clip_range


def clip_range_sym(x) -> ClipRange:
    """clipping.py:51-55."""
    rr = _row_search("sym", x)
    return ClipRange(float(rr.xmin[0].item()), float(rr.xmax[0].item()))


def clip_range_aciq(x, distribution: str = "laplacian", gaussian_constant: float | None = None) -> ClipRange:
    """clipping.py:115-139: alpha = constant * mean|x - mean| (5.03 for the laplacian
    assumption, the caller's gaussian_constant otherwise); alpha == 0 -> the data range."""
    if distribution == "laplacian":
        constant = 5.03
    elif distribution == "gaussian":
        if gaussian_constant is None:
            raise ValueError("gaussian clipping requires an explicit gaussian_constant; "
                             "only the laplacian constant is built in")
        constant = float(gaussian_constant)
    else:
        raise ValueError(f"distribution must be 'laplacian' or 'gaussian', got {distribution!r}")
    if not (np.isfinite(constant) and constant > 0.0):
        # alpha = constant * mad: zero (or negative) constants give the data range or an
        # inverted range in the reference; the device parameter is a positive constant
        if constant == 0.0:
            return clip_range_asym(x)
        raise ValueError(f"xmin exceeds xmax: gaussian_constant {constant} must be positive")
    rr = _row_search("aciq", x, param=constant)
    return ClipRange(float(rr.xmin[0].item()), float(rr.xmax[0].item()))


def clip_range_gss(x, nbits: int = 4, tol: float = 1e-4, counters: WorkCounters | None = None) -> ClipRange:
    """clipping.py:70-112: golden-section search of the symmetric threshold (4-bit objective;
    tol as given)."""
    if tol <= 0:
        raise ValueError(f"tol must be positive, got {tol}")
    if nbits not in (4, 8):
        raise ValueError(f"nbits must be 4 or 8, got {nbits}")
    if nbits != 4:
        raise ValueError("gss with nbits=8 is not on the B200 hot path (4-bit only)")
    rr = _row_search("gss", x, param=float(tol))
    _apply_counters(counters, "gss", 0, rr)
    return ClipRange(float(rr.xmin[0].item()), float(rr.xmax[0].item()))


def clip_range_table(table) -> ClipRange:
    """clipping.py:64-67: one (min, max) range over the whole table."""
    if not isinstance(table, EmbeddingTable):
        table = EmbeddingTable(table)
    _, rr = quantize_pack_table4(table, "table", "fp32", with_rows=True)
    return ClipRange(float(rr.xmin[0].item()), float(rr.xmax[0].item()))


def row_clip_range(method: str, x, nbits: int = 4, b: int = 200, r: float = 0.16,
                   counters: WorkCounters | None = None) -> ClipRange:
    """methods.py:43-60 for the GPU methods."""
    if method == "sym":
        return clip_range_sym(x)
    if method == "asym":
        return clip_range_asym(x)
    if method == "gss":
        return clip_range_gss(x, nbits, counters=counters)
    if method == "aciq":
        return clip_range_aciq(x)
    if method == "greedy":
        return clip_range_greedy(x, nbits, b, r, counters=counters)
    if method == "hist-brute":
        return clip_range_hist_brute(x, b, counters=counters)
    if method == "hist-apprx":
        return clip_range_hist_apprx(x, b, counters=counters)
    raise ValueError(f"{method!r} is not a row-wise uniform strategy")     # methods.py:60


def quant_mse_rows(x, xmin, xmax):
    """Per-row bit-exact quant_mse (table.py:81-103) of a CUDA table, 4-bit."""
    x = x.float().contiguous()
    rows, d = x.shape
    lo = torch.as_tensor(xmin, dtype=torch.float64, device=x.device).contiguous()
    hi = torch.as_tensor(xmax, dtype=torch.float64, device=x.device).contiguous()
    out = torch.empty(rows, dtype=torch.float64, device=x.device)
    _lib.check(_lib.load().eq4_quant_mse(_vp(x), rows, d, d, _vp(lo), _vp(hi), _vp(out),
                                         _stream_handle()))
    return out


def quant_mse(x, clip_range: ClipRange, nbits: int) -> float:
    """table.py:81-103 on the GPU (eq4_quant_mse_rows): float32 or float64 values, nbits 4
    or 8, numpy's pairwise float64 sum -- bit-exact."""
    if nbits not in (4, 8):
        raise ValueError(f"nbits must be 4 or 8, got {nbits}")
    flat = x.reshape(-1) if _is_cuda(x) else np.asarray(x).reshape(-1)
    n = int(flat.numel() if _is_cuda(x) else flat.size)
    if n == 0:
        return 0.0   # np.sum of an empty array
    t, f64 = _rows_on_device(flat)
    lo = torch.tensor([float(clip_range.xmin)], dtype=torch.float64, device=t.device)
    hi = torch.tensor([float(clip_range.xmax)], dtype=torch.float64, device=t.device)
    out = torch.empty(1, dtype=torch.float64, device=t.device)
    _lib.check(_lib.load().eq4_quant_mse_rows(_vp(t), int(f64), 1, n, n, _vp(lo), _vp(hi), int(nbits),
                                              _vp(out), _stream_handle()))
    return float(out.item())
