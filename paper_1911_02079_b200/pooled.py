"""Pooled lookup over packed 4-bit rows (SparseLengthsSum), SURVEY.md §8f item 1.

Drop-in for the reference's ``packed.PooledQuery`` / ``packed.sparse_lengths_sum_4bit``
(packed.py:122-177) and ``bench.bytes_per_pooled_row`` (bench.py:31-42).  The sum runs
in libeq4.so (``eq4_sparse_lengths_sum4``, csrc/eq4_sls.cu) on the GPU; results are
bit-identical to the reference's scalar ``sparse_lengths_sum_ref`` (packed.py:202-221):
float32 ``scale * code + bias`` rows accumulated in query order from 0.0.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .api import PackedTable4, _is_cuda, _stream_handle, _vp, packed_row_stride

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

DATA_TYPES = ("fp32", "int8", "int4")


def bytes_per_pooled_row(data_type: str, dim: int, aux_precision: str = "fp32") -> int:
    """Bytes read to dequantize one row under the fused layouts (bench.py:31-42)."""
    if dim < 1:
        raise ValueError(f"dim must be >= 1, got {dim}")
    if data_type == "fp32":
        return 4 * dim
    ab = 2 if aux_precision == "fp16" else 4
    if data_type == "int8":
        return dim + 2 * ab
    if data_type == "int4":
        return (dim + 1) // 2 + 2 * ab
    raise ValueError(f"data_type must be one of {DATA_TYPES}, got {data_type!r}")


class PooledQuery:
    """A batch of pooled lookups: indices, segmented by lengths (packed.py:122-144).

    Host arrays are validated here with the reference's messages; CUDA tensors stay
    on the device and are validated by the lookup kernel (same messages, raised by
    ``sparse_lengths_sum_4bit``)."""

    def __init__(self, indices, lengths):
        self.on_device = _is_cuda(indices) or _is_cuda(lengths)
        if self.on_device:
            dev = indices.device if _is_cuda(indices) else lengths.device
            self.indices = torch.as_tensor(indices).to(dev, torch.int64).reshape(-1).contiguous()
            self.lengths = torch.as_tensor(lengths).to(dev, torch.int64).reshape(-1).contiguous()
            return
        self.indices = np.asarray(indices, dtype=np.int64).ravel()
        self.lengths = np.asarray(lengths, dtype=np.int64).ravel()
        if np.any(self.lengths < 0):
            raise ValueError("lengths must be non-negative")
        if int(self.lengths.sum()) != self.indices.size:
            raise ValueError(
                f"lengths sum to {int(self.lengths.sum())} but there are {self.indices.size} indices")

    @property
    def batch(self) -> int:
        return int(self.lengths.numel() if self.on_device else self.lengths.size)


def sparse_lengths_sum_4bit(p: PackedTable4, query: PooledQuery, *, out=None, stream=None,
                            check: bool = True):
    """out[s] = sum of the dequantized rows of segment s (packed.py:167-177).

    Returns a float32 numpy array (batch, dim) for a host query, or a CUDA tensor for a
    device query (``out`` may be a preallocated CUDA tensor).  ``check=False`` skips the
    host synchronisation that turns device status bits into the reference's exceptions.
    """
    if not isinstance(p, PackedTable4):
        raise TypeError(f"expected a PackedTable4, got {type(p).__name__}")
    if not isinstance(query, PooledQuery):
        query = PooledQuery(*query)
    L = _lib.load()
    packed = p.to_device()
    dev = packed.device
    if stream is not None and stream != torch.cuda.current_stream(dev):
        # allocate, launch and read the status word on the caller's stream
        with torch.cuda.stream(stream):
            return sparse_lengths_sum_4bit(p, query, out=out, stream=None, check=check)
    idx = query.indices if query.on_device else torch.from_numpy(query.indices).to(dev)
    ln = query.lengths if query.on_device else torch.from_numpy(query.lengths).to(dev)
    batch, nidx = int(ln.numel()), int(idx.numel())
    if out is None:
        out = torch.empty((batch, p.dim), dtype=torch.float32, device=dev)
    elif not (_is_cuda(out) and out.dtype == torch.float32 and out.is_contiguous()
              and out.numel() == batch * p.dim):
        raise ValueError(f"out must be a contiguous CUDA float32 tensor of {batch}x{p.dim}")
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.check(L.eq4_sparse_lengths_sum4(
        _vp(packed), p.rows, p.dim, _lib.AUX[p.aux_precision], _vp(idx) if nidx else None, nidx,
        _vp(ln) if batch else None, batch, _vp(out) if batch else None, _vp(status), _vp(bad),
        _stream_handle(stream)))
    if check:
        st = int(status.item())
        if st & _lib.STATUS_QUERY:
            if bool((ln < 0).any()):
                raise ValueError("lengths must be non-negative")
            raise ValueError(f"lengths sum to {int(ln.sum())} but there are {nidx} indices")
        if st & _lib.STATUS_INDEX:
            pos = int(bad.item())
            raise IndexError(f"query index {int(idx[pos])} at position {pos} out of range for "
                             f"{p.rows} rows")
    if query.on_device:
        return out
    return out.cpu().numpy()


__all__ = ["DATA_TYPES", "PooledQuery", "bytes_per_pooled_row", "sparse_lengths_sum_4bit",
           "packed_row_stride"]
