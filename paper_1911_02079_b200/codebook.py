"""Row-wise 16-value codebooks (KMEANS), SURVEY.md §8f item 4.

Mirror of the reference's ``codebook`` row-wise path (codebook.py:35-172):
``quantize_table_kmeans`` / ``quantize_row_kmeans`` return a ``CodebookQuantTable``
whose codebooks and indices are bit-identical to the reference's.  The Lloyd
iterations run in libeq4.so (``eq4_kmeans_rows``), one GPU lane per row, and write
the EMBQ kmeans_row payload (sorted codebook + nibble-packed indices per row), which
``fileio.write_embq`` stores verbatim.  The two-tier ``kmeans-cls`` scheme is not on
the GPU path.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .api import EmbeddingTable, _check_aux, _is_cuda, _stream_handle, _vp

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

CODEBOOK_SIZE = 16
_AUX_NP = {"fp32": np.float32, "fp16": np.float16}


def kmeans_row_stride(dim: int, aux_precision: str) -> int:
    """Bytes of one kmeans_row EMBQ record (fileio.py:105-110)."""
    return CODEBOOK_SIZE * (2 if aux_precision == "fp16" else 4) + (dim + 1) // 2


class CodebookRowQuant:
    """One row against its own sorted 16-value codebook (codebook.py:120-129)."""

    def __init__(self, codebook, indices):
        self.codebook = codebook
        self.indices = indices

    def dequantize(self) -> np.ndarray:
        return self.codebook.astype(np.float32)[self.indices]


class CodebookQuantTable:
    """Per-row codebooks for a whole table (codebook.py:140-161)."""

    def __init__(self, codebooks, indices, aux_precision: str = "fp32"):
        self.codebooks = codebooks
        self.indices = indices
        self.aux_precision = aux_precision

    @property
    def rows(self) -> int:
        return self.indices.shape[0]

    @property
    def dim(self) -> int:
        return self.indices.shape[1]

    def row(self, i: int) -> CodebookRowQuant:
        return CodebookRowQuant(self.codebooks[i], self.indices[i])

    def dequantize(self) -> np.ndarray:
        out = self.codebooks.astype(np.float32)
        return np.take_along_axis(out, self.indices.astype(np.int64), axis=1)

    @classmethod
    def from_payload(cls, payload, rows: int, dim: int, aux_precision: str) -> "CodebookQuantTable":
        """Decode EMBQ kmeans_row records (fileio.py:156-163)."""
        ab = 2 if aux_precision == "fp16" else 4
        fused = np.asarray(payload, dtype=np.uint8).reshape(rows, kmeans_row_stride(dim, aux_precision))
        books = np.ascontiguousarray(fused[:, : CODEBOOK_SIZE * ab]).view(
            "<f2" if ab == 2 else "<f4").reshape(rows, CODEBOOK_SIZE)
        nib = fused[:, CODEBOOK_SIZE * ab:]
        idx = np.empty((rows, 2 * nib.shape[1]), np.uint8)
        idx[:, 0::2] = nib & 0x0F
        idx[:, 1::2] = nib >> 4
        t = cls(books.astype(_AUX_NP[aux_precision]), np.ascontiguousarray(idx[:, :dim]), aux_precision)
        t._payload = np.ascontiguousarray(fused).reshape(-1)
        return t

    def payload(self) -> np.ndarray:
        """The EMBQ kmeans_row records of this table (books then nibbles per row)."""
        p = getattr(self, "_payload", None)
        if p is not None:
            return p
        ab = 2 if self.aux_precision == "fp16" else 4
        books = np.ascontiguousarray(self.codebooks.astype(_AUX_NP[self.aux_precision])).view(
            np.uint8).reshape(self.rows, CODEBOOK_SIZE * ab)
        idx = self.indices
        if self.dim % 2:
            idx = np.concatenate([idx, np.zeros((self.rows, 1), np.uint8)], axis=1)
        nib = (idx[:, 0::2] | (idx[:, 1::2] << 4)).astype(np.uint8)
        return np.concatenate([books, nib], axis=1).reshape(-1)


def kmeans_rows(x, aux_precision: str = "fp32", *, out=None, iters=None, stream=None, check=True):
    """Run the row-wise KMEANS kernel on a CUDA fp32 table; returns the kmeans_row payload
    (CUDA uint8 tensor, rows x kmeans_row_stride)."""
    _check_aux(aux_precision)
    x = x.float().contiguous()
    rows, d = x.shape
    stride = kmeans_row_stride(d, aux_precision)
    if out is None:
        out = torch.empty(rows * stride, dtype=torch.uint8, device=x.device)
    status = torch.zeros(1, dtype=torch.int32, device=x.device)
    _lib.check(_lib.load().eq4_kmeans_rows(_vp(x), rows, d, d, _lib.AUX[aux_precision], _vp(out),
                                            _vp(iters), _vp(status), _stream_handle(stream)))
    if check and int(status.item()) & _lib.STATUS_NONFINITE:
        raise ValueError("table contains non-finite values (NaN/Inf)")
    return out


def quantize_table_kmeans(table, aux_precision: str = "fp32") -> CodebookQuantTable:
    """codebook.py:164-172 on the GPU."""
    _check_aux(aux_precision)
    if not isinstance(table, EmbeddingTable):
        table = EmbeddingTable(table)
    if table.on_device:
        x = table._device
    else:
        x = torch.from_numpy(np.ascontiguousarray(table.values)).cuda()
    payload = kmeans_rows(x, aux_precision).cpu().numpy()
    return CodebookQuantTable.from_payload(payload, table.rows, table.dim, aux_precision)


def quantize_row_kmeans(x, aux_precision: str = "fp32") -> CodebookRowQuant:
    """codebook.py:108-123 (default max_iter / tol)."""
    a = np.asarray(x, dtype=np.float64).ravel()
    if a.size == 0:
        raise ValueError("input vector is empty")
    t = quantize_table_kmeans(EmbeddingTable(a.astype(np.float32).reshape(1, -1)), aux_precision)
    return t.row(0)


__all__ = ["CODEBOOK_SIZE", "CodebookRowQuant", "CodebookQuantTable", "kmeans_row_stride",
           "kmeans_rows", "quantize_table_kmeans", "quantize_row_kmeans"]
