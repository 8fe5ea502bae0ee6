"""Row sharding of a table across ranks (one process per GPU).

Rows are independent (methods.py:86-88: the reference quantizes row by row;
SPEC.md: "a table-level driver may process rows concurrently"), so N GPUs take
contiguous row ranges and no collective is needed on the data path.  The only
optional exchange is an all-gather of the packed shards (fixed row stride, so
the shards concatenate into the reference's PackedTable4 buffer).
"""

from __future__ import annotations

from typing import Callable

import numpy as np


def shard_bounds(rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) of `rank` (the first rows % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(rows, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a scalar over all ranks (step times are reported as the slowest rank's)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_packed(local: "torch.Tensor", rows: int, stride: int, group=None) -> "torch.Tensor":
    """All-gather the ranks' packed shards (1-D uint8, rows_local * stride bytes) in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [shard_bounds(rows, r, world) for r in range(world)]
    maxb = max(stop - start for start, stop in sizes) * stride
    buf = torch.zeros(maxb, dtype=torch.uint8, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[r][: (stop - start) * stride] for r, (start, stop) in enumerate(sizes)])


def quantize_pack_sharded(table, method: str, aux_precision: str = "fp16", b: int = 200,
                          r: float = 0.16, *, group=None, gather: bool = True,
                          compute: Callable | None = None, table_range: Callable | None = None,
                          compute_range: Callable | None = None):
    """Quantize this rank's row range of `table`; optionally all-gather the packed table.

    Every row-wise method is independent per row.  TABLE (clipping.py:64-67) is not: its
    one range spans the whole table, so the ranks' shard ranges are combined first (an
    all-reduce of min and max -- the only collective on this path) and every shard is
    quantized against that global range.

    ``compute(rows_array, method, aux, b, r) -> uint8 tensor`` defaults to the B200 path
    (quantize_pack_table4 on this rank's GPU); ``table_range(rows_array) -> (lo, hi)``
    and ``compute_range(rows_array, lo, hi, aux) -> uint8 tensor`` (TABLE only) default
    to libeq4.so as well.  Tests inject CPU functions to exercise the orchestration over
    gloo.
    """
    import torch
    import torch.distributed as dist

    from .api import packed_row_stride

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    rows = int(table.shape[0])
    start, stop = shard_bounds(rows, rank, world)
    stride = packed_row_stride(int(table.shape[1]), aux_precision)

    def on_gpu(x):
        if not (isinstance(x, torch.Tensor) and x.is_cuda):
            x = torch.as_tensor(np.ascontiguousarray(x)).cuda()
        return x

    if compute is None:
        from .api import quantize_pack_table4

        def compute(x, m, a, bb, rr):
            return quantize_pack_table4(on_gpu(x), m, a, bb, rr)[0].device_buffer

    if method == "table":
        if table_range is None:
            from .api import quantize_pack_table4

            def table_range(x):   # the shard's own TABLE range from the device kernels
                _, rr = quantize_pack_table4(on_gpu(x), "table", aux_precision, with_rows=True)
                return float(rr.xmin[0].item()), float(rr.xmax[0].item())
        if compute_range is None:
            def compute_range(x, lo, hi, aux):   # quantize_table_uniform against (lo, hi), packed
                from .codec import _quantize_rows

                t = on_gpu(x).float().contiguous()
                codes, sc, bi = _quantize_rows(t, False, [lo], [hi], 4, aux)
                return _pack_device(codes, sc, bi, aux)
        local_x = table[start:stop]
        lo, hi = table_range(local_x) if stop > start else (np.inf, -np.inf)
        if world > 1:
            dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
                else torch.device("cpu")
            lh = torch.tensor([lo, -hi], dtype=torch.float64, device=dev)
            dist.all_reduce(lh, op=dist.ReduceOp.MIN, group=group)
            lo, hi = float(lh[0].item()), -float(lh[1].item())
        local = compute_range(local_x, lo, hi, aux_precision)
    else:
        local = compute(table[start:stop], method, aux_precision, b, r)
    if not gather or world == 1:
        return local
    return gather_packed(local, rows, stride, group)


def _pack_device(codes, sc, bi, aux):
    """pack_table4 of device codes / scales / biases (eq4_pack) -> packed device buffer."""
    import torch

    from . import _lib
    from .api import _stream_handle, _vp, packed_row_stride

    rows, d = int(codes.shape[0]), int(codes.shape[1])
    out = torch.empty(rows * packed_row_stride(d, aux), dtype=torch.uint8, device=codes.device)
    _lib.check(_lib.load().eq4_pack(_vp(codes), rows, d, _lib.AUX[aux], _vp(sc), _vp(bi), _vp(out),
                                    _stream_handle()))
    return out
