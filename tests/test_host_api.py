"""CPU tests: the C ABI library loads and exports include/eq4.h, the host API mirrors the
reference's validation and error texts, and the multi-rank row-sharding path (gloo)."""

import os
import re
import socket

import numpy as np
import pytest

import oracle
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import _lib
from paper_1911_02079_b200.sharding import shard_bounds

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "eq4.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(eq4_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = eq.load()
    declared = _header_functions()
    assert declared == sorted(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.eq4_version().decode().startswith("eq4")


def test_packed_row_stride_matches_reference_kats():
    # test_packed.py:212-215 and packed.py:32-33
    assert eq.packed_row_stride(128, "fp32") == 72
    assert eq.packed_row_stride(128, "fp16") == 68
    assert eq.packed_row_stride(7, "fp32") == 12
    L = eq.load()
    for d in (1, 7, 64, 129, 2048):
        for aux in ("fp16", "fp32"):
            assert L.eq4_packed_row_stride(d, _lib.AUX[aux]) == eq.packed_row_stride(d, aux)
            assert oracle.packed_row_stride(d, aux) == eq.packed_row_stride(d, aux)


def test_c_abi_rejects_bad_arguments_before_any_launch():
    L = eq.load()
    # rows < 1 / null buffers / bad aux / bad b / bad r: EQ4_EINVAL with a message, no CUDA call
    assert L.eq4_quantize_pack(None, 0, 4, 4, 1, 200, 0.16, 1, None, None, None, None, None, None,
                               None, None) == _lib.EQ4_EINVAL
    assert "at least 1x1" in _lib.last_error()
    dummy = np.zeros(4, np.float32)
    out = np.zeros(16, np.uint8)
    p = dummy.ctypes.data_as(__import__("ctypes").c_void_p)
    o = out.ctypes.data_as(__import__("ctypes").c_void_p)
    assert L.eq4_quantize_pack(p, 1, 4, 4, 1, 0, 0.16, 1, o, None, None, None, None, None, None,
                               None) == _lib.EQ4_EINVAL
    assert _lib.last_error() == "b must be >= 1, got 0"
    assert L.eq4_quantize_pack(p, 1, 4, 4, 1, 200, 1.5, 1, o, None, None, None, None, None, None,
                               None) == _lib.EQ4_EINVAL
    assert _lib.last_error().startswith("r must be in (0, 1]")
    assert L.eq4_quantize_pack(p, 1, 4, 4, 1, 200, 0.16, 7, o, None, None, None, None, None, None,
                               None) == _lib.EQ4_EINVAL


@pytest.mark.parametrize("kw,msg", [
    (dict(method="nope"), "unknown method 'nope'"),
    (dict(method="kmeans", nbits=8), "kmeans is 4-bit only, got nbits=8"),
    (dict(method="greedy", k=3), "k applies only to kmeans-cls, not greedy"),
])
def test_quantize_table_validation_matches_reference(kw, msg, ref):
    t = np.ones((2, 4), np.float32)
    with pytest.raises(ValueError) as ours:
        eq.quantize_table(t, **kw)
    with pytest.raises(ValueError) as theirs:
        ref.quantize_table(ref.EmbeddingTable(t), **kw)
    assert str(ours.value) == str(theirs.value)
    assert msg in str(ours.value)


def test_greedy_parameter_errors_match_reference(ref):
    x = [1.0, 2.0]
    for kw in (dict(b=0), dict(r=0.0), dict(r=1.5)):
        with pytest.raises(ValueError) as theirs:
            ref.clip_range_greedy(x, 4, **kw)
        with pytest.raises(ValueError) as ours:
            eq.clip_range_greedy(x, 4, **kw)
        assert str(ours.value) == str(theirs.value)


def test_methods_off_the_hot_path_raise_instead_of_falling_back():
    t = np.ones((2, 4), np.float32)
    for m in ("kmeans-cls",):
        with pytest.raises(ValueError, match="not on the B200 hot path"):
            eq.quantize_table(t, m)
    with pytest.raises(ValueError, match="not on the B200 hot path"):
        eq.quantize_table(t, "greedy", nbits=8)


def test_containers_mirror_reference():
    # table.py:22-31, test_table.py:11-47
    t = eq.EmbeddingTable(np.array([[1, 2, 3], [4, 5, 6]], dtype=np.float32))
    assert t.row(0).tolist() == [1, 2, 3] and (t.rows, t.dim) == (2, 3)
    with pytest.raises(IndexError):
        t.row(2)
    with pytest.raises(ValueError, match="non-finite"):
        eq.EmbeddingTable(np.array([[1.0, np.nan]], dtype=np.float32))
    with pytest.raises(ValueError):
        eq.EmbeddingTable(np.zeros((0, 4), dtype=np.float32))
    with pytest.raises(ValueError):
        t.values[0, 0] = 5.0
    with pytest.raises(ValueError):
        eq.ClipRange(1.0, -1.0)
    with pytest.raises(ValueError):
        eq.ClipRange(0.0, np.inf)
    c = eq.WorkCounters(1, 2, 3)
    c.merge(eq.WorkCounters(1, 1, 1))
    assert (c.loss_evals, c.candidate_evals, c.bin_visits) == (2, 3, 4)


def test_uniform_quant_table_validation():
    with pytest.raises(ValueError):
        eq.UniformQuantTable(np.zeros(4, np.uint8), [1.0], [0.0], 4)
    with pytest.raises(ValueError):
        eq.UniformQuantTable(np.zeros((2, 4), np.uint8), [1.0], [0.0], 4)
    q = eq.UniformQuantTable(np.zeros((1, 4), np.uint8), [1.0], [0.0], 8)
    with pytest.raises(ValueError, match="4-bit"):
        eq.pack_table4(q)


def test_shard_bounds_cover_rows_exactly():
    for rows in (1, 7, 64, 1000, 20_000_001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(rows, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded_worker(rank, world, port, x, q):
    import torch
    import torch.distributed as dist

    from paper_1911_02079_b200.sharding import max_over_ranks, quantize_pack_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def cpu_compute(rows, method, aux, b, r):   # the orchestration under test, CPU compute
            return torch.from_numpy(oracle.quantize_pack_table(rows, method, b, r, aux).packed)

        full = quantize_pack_sharded(x, "greedy", "fp16", compute=cpu_compute)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((full.numpy().tobytes(), t))
    finally:
        dist.destroy_process_group()


def test_row_sharded_quantization_over_gloo():
    import torch.multiprocessing as mp

    from oracle import rng

    x = rng.mixed_table(1001, 64, 3)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, x, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.quantize_pack_table(x, "greedy", 200, 0.16, "fp16").packed
    assert got == want.tobytes()
    assert tmax == float(world)


def _sharded_table_worker(rank, world, port, x, q):
    import torch
    import torch.distributed as dist

    from paper_1911_02079_b200.sharding import quantize_pack_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def cpu_range(rows):          # the shard's own min / max (the oracle's TABLE range)
            t = oracle.quantize_pack_table(rows, "table", aux="fp16")
            return float(t.xmin[0]), float(t.xmax[0])

        def cpu_quantize(rows, lo, hi, aux):   # quantize_table_uniform against one ClipRange
            rows = np.ascontiguousarray(rows, np.float32)
            out = []
            for row in rows:
                c, s, b = oracle.quantize_uniform(row, lo, hi, 4, aux)
                out.append(oracle.pack_table4(c[None], [s], [b], aux))
            return torch.from_numpy(np.concatenate(out))

        full = quantize_pack_sharded(x, "table", "fp16", table_range=cpu_range, compute_range=cpu_quantize)
        if rank == 0:
            q.put(full.numpy().tobytes())
    finally:
        dist.destroy_process_group()


def test_row_sharded_table_uses_the_global_range_over_gloo():
    """TABLE (clipping.py:64-67) spans the whole table: the shards all-reduce their ranges and
    quantize against the global one -- the gathered bytes equal the unsharded oracle's."""
    import torch.multiprocessing as mp

    from oracle import rng

    x = rng.mixed_table(301, 24, 9)
    x[5, 3] = 40.0        # the global max sits in rank 0's shard,
    x[250, 7] = -35.0     # the global min in rank 1's
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_table_worker, args=(r, world, port, x, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == oracle.quantize_pack_table(x, "table", aux="fp16").packed.tobytes()


def test_pooled_query_validation_matches_reference(ref):
    from embquant.packed import PooledQuery as RefQuery

    for i, l in (([1, 2], [1]), ([1], [-1, 2]), ([], [0, -1])):
        with pytest.raises(ValueError) as theirs:
            RefQuery(i, l)
        with pytest.raises(ValueError) as ours:
            eq.PooledQuery(i, l)
        assert str(ours.value) == str(theirs.value)
    q = eq.PooledQuery([3, 1, 2], [2, 0, 1])
    assert q.batch == 3 and q.indices.dtype == np.int64


def test_bytes_per_pooled_row_kats():
    # test_packed.py:159-181
    assert eq.bytes_per_pooled_row("fp32", 128) == 512
    assert eq.bytes_per_pooled_row("int8", 128, "fp32") == 136
    assert eq.bytes_per_pooled_row("int4", 128, "fp32") == 72
    assert eq.bytes_per_pooled_row("int4", 128, "fp16") == 68
    with pytest.raises(ValueError):
        eq.bytes_per_pooled_row("int2", 8)


def test_row_clip_range_table_is_not_rowwise_like_reference(ref):
    x = [1.0, 2.0, 3.0]
    with pytest.raises(ValueError) as theirs:
        ref.row_clip_range("table", x)
    with pytest.raises(ValueError) as ours:
        eq.row_clip_range("table", x)
    assert str(ours.value) == str(theirs.value)
    with pytest.raises(ValueError) as theirs:
        ref.clip_range_gss(x, 4, tol=0.0)
    with pytest.raises(ValueError) as ours:
        eq.clip_range_gss(x, 4, tol=0.0)
    assert str(ours.value) == str(theirs.value)
    for kw in (dict(distribution="gaussian"), dict(distribution="cauchy")):
        with pytest.raises(ValueError) as theirs:
            ref.clip_range_aciq(x, **kw)
        with pytest.raises(ValueError) as ours:
            eq.clip_range_aciq(x, **kw)
        assert str(ours.value) == str(theirs.value)
