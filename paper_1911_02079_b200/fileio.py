"""EMBT / EMBQ containers on the hot path's input and output side.

Mirrors the reference's ``fileio`` (fileio.py:1-200) for float tables (EMBT) and the
uniform4 EMBQ container, with the same header layouts and ``DataError`` texts, plus
``quantize_file``: EMBT -> EMBQ streamed through the GPU by libeq4.so
(``eq4_quantize_file``: pinned chunks, H2D / kernel / D2H / disk write overlapped) so a
20M-row table never has to sit in host or device memory whole.  ``write_embq`` of a
device-resident PackedTable4 streams the packed rows out of HBM without a host repack.
"""

from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

from . import _lib
from .api import (ALL_METHODS, GPU_METHODS, EmbeddingTable, PackedTable4, UniformQuantTable,
                  _check_aux, _check_method_params, _vp, pack_table4, packed_row_stride)

__all__ = ["DataError", "read_embt", "write_embt", "read_embq", "write_embq", "quantize_file"]

_EMBT_MAGIC = b"EMBT"
_EMBQ_MAGIC = b"EMBQ"
_VERSION = 1
_EMBT_HEADER = struct.Struct("<4sIQQB")     # fileio.py:26
_EMBQ_HEADER = struct.Struct("<4sIBBQQ")    # fileio.py:27
_SCHEME_CODES = {"uniform4": 0, "uniform8": 1, "kmeans_row": 2, "kmeans_cls": 3}
_SCHEME_NAMES = {v: k for k, v in _SCHEME_CODES.items()}
_AUX_CODES = {"fp32": 0, "fp16": 1}
_AUX_NAMES = {v: k for k, v in _AUX_CODES.items()}


class DataError(ValueError):
    """Malformed or inconsistent data file (fileio.py:37-38)."""


def write_embt(path, table) -> None:
    """fileio.py:40-45."""
    if not isinstance(table, EmbeddingTable):
        table = EmbeddingTable(table)
    header = _EMBT_HEADER.pack(_EMBT_MAGIC, _VERSION, table.rows, table.dim, 0)
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(np.ascontiguousarray(table.values, dtype="<f4").tobytes())


def _embt_header(path, head: bytes, size: int):
    """Header checks of fileio.py:48-66 (same order and messages); returns (rows, dim)."""
    if size < _EMBT_HEADER.size:
        raise DataError(f"{path}: truncated header ({size} bytes)")
    magic, version, rows, dim, dtype = _EMBT_HEADER.unpack_from(head)
    if magic != _EMBT_MAGIC:
        raise DataError(f"{path}: bad magic {magic!r}")
    if version != _VERSION:
        raise DataError(f"{path}: unsupported version {version}")
    if dtype != 0:
        raise DataError(f"{path}: unsupported dtype code {dtype}")
    if rows < 1 or dim < 1:
        raise DataError(f"{path}: invalid shape {rows}x{dim}")
    expected = rows * dim * 4
    payload = size - _EMBT_HEADER.size
    if payload != expected:
        raise DataError(f"{path}: truncated payload ({payload} of {expected} bytes)")
    return rows, dim


def read_embt(path) -> EmbeddingTable:
    """fileio.py:48-70."""
    with open(path, "rb") as fh:
        blob = fh.read()
    rows, dim = _embt_header(path, blob[: _EMBT_HEADER.size], len(blob))
    values = np.frombuffer(blob, dtype="<f4", offset=_EMBT_HEADER.size).reshape(rows, dim)
    if not np.all(np.isfinite(values)):
        raise DataError(f"{path}: payload contains non-finite values")
    return EmbeddingTable(values)


def read_embq(path) -> PackedTable4:
    """fileio.py:130-164 for the uniform4 scheme (the hot path's output format)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _EMBQ_HEADER.size:
        raise DataError(f"{path}: truncated header ({len(blob)} bytes)")
    magic, version, scheme_code, aux_code, rows, dim = _EMBQ_HEADER.unpack_from(blob)
    if magic != _EMBQ_MAGIC:
        raise DataError(f"{path}: bad magic {magic!r}")
    if version != _VERSION:
        raise DataError(f"{path}: unsupported version {version}")
    if scheme_code not in _SCHEME_NAMES:
        raise DataError(f"{path}: unknown scheme code {scheme_code}")
    if aux_code not in _AUX_NAMES:
        raise DataError(f"{path}: unknown aux code {aux_code}")
    if rows < 1 or dim < 1:
        raise DataError(f"{path}: invalid shape {rows}x{dim}")
    scheme = _SCHEME_NAMES[scheme_code]
    aux = _AUX_NAMES[aux_code]
    if scheme == "kmeans_row":                                 # fileio.py:156-163
        from .codebook import CodebookQuantTable, kmeans_row_stride

        nbytes = rows * kmeans_row_stride(dim, aux)
        if len(blob) - _EMBQ_HEADER.size < nbytes:
            raise DataError(f"{path}: truncated payload (codebook rows)")
        if len(blob) - _EMBQ_HEADER.size != nbytes:
            raise DataError(f"{path}: payload size mismatch")
        return CodebookQuantTable.from_payload(
            np.frombuffer(blob, dtype=np.uint8, offset=_EMBQ_HEADER.size), rows, dim, aux)
    if scheme != "uniform4":
        raise ValueError(f"EMBQ scheme {scheme!r} is not on the B200 hot path (uniform4, kmeans_row)")
    nbytes = rows * packed_row_stride(dim, aux)
    if len(blob) - _EMBQ_HEADER.size < nbytes:
        raise DataError(f"{path}: truncated payload (packed rows)")
    if len(blob) - _EMBQ_HEADER.size != nbytes:
        raise DataError(f"{path}: payload size mismatch")
    return PackedTable4(rows, dim, aux, np.frombuffer(blob, dtype=np.uint8, offset=_EMBQ_HEADER.size).copy())


def write_embq(path, quant) -> None:
    """fileio.py:94-101 for 4-bit uniform tables: header + PackedTable4 bytes verbatim.
    A device-resident PackedTable4 is streamed out of HBM by the native writer."""
    from .codebook import CodebookQuantTable

    if isinstance(quant, CodebookQuantTable):                  # fileio.py:105-110
        head = _EMBQ_HEADER.pack(_EMBQ_MAGIC, _VERSION, _SCHEME_CODES["kmeans_row"],
                                 _AUX_CODES[quant.aux_precision], quant.rows, quant.dim)
        with open(path, "wb") as fh:
            fh.write(head)
            fh.write(quant.payload().tobytes())
        return
    if isinstance(quant, UniformQuantTable):
        if quant.nbits != 4:
            raise ValueError("8-bit EMBQ (uniform8) is not on the B200 hot path")
        quant = pack_table4(quant)
    if not isinstance(quant, PackedTable4):
        raise TypeError(f"cannot serialize {type(quant).__name__}")
    L = _lib.load()
    aux = _lib.AUX[quant.aux_precision]
    if quant._buffer is None and quant.device_buffer is not None:
        rc = L.eq4_write_embq(os.fsencode(path), _vp(quant.device_buffer), quant.rows, quant.dim,
                              aux, 1)
    else:
        buf = np.ascontiguousarray(quant.buffer)
        rc = L.eq4_write_embq(os.fsencode(path), _vp(buf), quant.rows, quant.dim, aux, 0)
    _lib.check(rc)


def quantize_file(in_path, out_path, method: str, aux_precision: str = "fp32", b: int = 200,
                  r: float = 0.16, chunk_rows: int = 0) -> None:
    """write_embq(out, quantize_table(read_embt(in), method, 4, aux, b, r)), streamed on the GPU.

    Same validation and messages as the reference's read_embt / quantize_table; a
    non-finite payload raises read_embt's DataError and leaves no output file."""
    if method not in ALL_METHODS:
        raise ValueError(f"unknown method {method!r}; expected one of {ALL_METHODS}")
    if method == "kmeans":                                     # codebook.py:164-172, kmeans_row
        from .codebook import quantize_table_kmeans

        write_embq(out_path, quantize_table_kmeans(read_embt(in_path), aux_precision))
        return
    if method not in GPU_METHODS:
        raise ValueError(f"{method!r} with nbits=4 is not on the B200 hot path "
                         f"(supported: {GPU_METHODS} at nbits=4)")
    _check_aux(aux_precision)
    _check_method_params(method, b, r)
    size = os.path.getsize(in_path)
    with open(in_path, "rb") as fh:
        head = fh.read(_EMBT_HEADER.size)
    _embt_header(in_path, head, size)
    L = _lib.load()
    bad = np.full(1, -1, np.int64)
    lohi = np.zeros(2)
    rc = L.eq4_quantize_file(os.fsencode(in_path), os.fsencode(out_path), _lib.METHOD[method], int(b),
                             float(r), _lib.AUX[aux_precision], int(chunk_rows),
                             bad.ctypes.data_as(ctypes.c_void_p), lohi.ctypes.data_as(ctypes.c_void_p))
    if rc == _lib.EQ4_EDATA:
        raise DataError(_lib.last_error())
    if rc == _lib.EQ4_ERANGE:
        raise ValueError(f"xmin {float(lohi[0])} exceeds xmax {float(lohi[1])}")
    _lib.check(rc)
