"""GREEDY on wide vector rows (d >= 1024): the table walk k_greedy_table (eq4_gtable.cuh) --
histogram of the row into half-unit bins of the candidate grid, suffix scan to
chi(T) = sum max(y - T, 0), 15 table reads per candidate -- in place of the per-element
screen k_greedy_fast.  Bytes, float64 ranges, iteration counts and best pairs must equal the
oracle's (clipping.py:142-193, table.py:81-103, uniform.py:60-80, packed.py:32-83) and the
per-element screen's (development switch EQ4_DEV_TABLE_MIN_D moves the dispatch threshold)."""

import os

import numpy as np
import pytest

import oracle
from oracle import rng
from test_oracle_golden import _bits

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _run(x, aux="fp16", b=200, r=0.16, min_d=None):
    import paper_1911_02079_b200 as eq
    from paper_1911_02079_b200 import _lib

    if min_d is not None:
        os.environ["EQ4_DEV_TABLE_MIN_D"] = str(min_d)
    try:
        _lib.diag_counters(reset=True)
        p, rr = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "greedy", aux, b, r, with_rows=True)
        torch.cuda.synchronize()
        diag = _lib.diag_counters(reset=True)
    finally:
        os.environ.pop("EQ4_DEV_TABLE_MIN_D", None)
    return p, rr, diag


def _check(x, aux="fp16", b=200, r=0.16, min_d=None):
    import paper_1911_02079_b200 as eq

    p, rr, diag = _run(x, aux, b, r, min_d)
    want = oracle.quantize_pack_table(x, "greedy", b, r, aux)
    st = eq.packed_row_stride(x.shape[1], aux)
    bad = np.nonzero((p.buffer.reshape(-1, st) != want.packed.reshape(-1, st)).any(1))[0]
    assert bad.size == 0, (x.shape, aux, b, r, bad[:8])
    assert np.array_equal(_bits(rr.xmin.cpu().numpy()), _bits(want.xmin))
    assert np.array_equal(_bits(rr.xmax.cpu().numpy()), _bits(want.xmax))
    assert np.array_equal(rr.info0.cpu().numpy(), want.info0)
    return p, rr, diag


@pytest.mark.parametrize("d", [1024, 1028, 1500, 2048, 3000, 4096, 6000, 8192, 12344, 16384])
def test_table_walk_vs_oracle(d):
    rows = max(24, 400_000 // d)
    x = rng.mixed_table(rows, d, d) if d % 8 else rng.sample_table("gaussian", 0.0, 1.0, d, rows, d)
    _, _, diag = _check(x, "fp16" if d % 3 else "fp32", min_d=16)
    assert diag["deferred_rows"] <= rows // 20, diag   # generic rows stay in the table walk


@pytest.mark.parametrize("b,r", [(8, 1.0), (40, 0.5), (64, 0.16), (200, 0.9), (333, 0.16), (400, 0.3)])
def test_table_walk_b_and_r(b, r):
    """Table sizes from 242 to 12,002 bins; r = 1.0 walks until the candidate range inverts
    (the reference's ValueError rows are reported by the exact kernel)."""
    x = rng.mixed_table(96, 1536, 5 * b)
    if r == 1.0:
        import paper_1911_02079_b200 as eq
        try:
            want = oracle.quantize_pack_table(x, "greedy", b, r, "fp16")
        except ValueError:
            with pytest.raises(ValueError):
                eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "greedy", "fp16", b, r)
            return
    _check(x, "fp16", b, r, min_d=16)


def test_table_walk_equals_per_element_screen():
    """Same table through both screens (dispatch threshold moved): identical outputs."""
    x = rng.mixed_table(3000, 1024, 99)
    p0, r0, d0 = _run(x, min_d=1024)
    p1, r1, d1 = _run(x, min_d=1 << 20)
    assert np.array_equal(p0.buffer, p1.buffer)
    for f in ("xmin", "xmax", "info0", "info1"):
        assert torch.equal(getattr(r0, f), getattr(r1, f)), f
    assert d0["deferred_rows"] < d1["deferred_rows"], (d0, d1)   # the narrower band defers fewer rows


def test_table_walk_narrow_rows_forced():
    """The table walk forced onto narrow rows (d = 64, 128, 256): still the oracle's bytes."""
    for d in (64, 128, 256):
        x = rng.mixed_table(4000, d, d + 1)
        _check(x, "fp16", min_d=16)


def test_table_walk_crafted_rows():
    """Rows the walk hands over (zero min / max, constant, non-finite-free coarse grid), exact
    L/R ties (symmetric rows), grid-valued rows with many elements on thresholds, repeated
    values, rows with most mass in one bin."""
    d = 2048
    g = np.random.default_rng(5)
    rows = []
    base = rng.mixed_table(16, d, 3)
    r0 = np.abs(base[0]); r0[3] = 0.0; rows.append(r0)                       # zero minimum
    r1 = -np.abs(base[1]); r1[1] = 0.0; rows.append(r1)                      # zero maximum
    rows.append(np.full(d, 1.25, np.float32))                                # constant
    rows.append((base[2] * 1e-9 + 3e4).astype(np.float32))                   # coarse reference grid
    h = np.abs(base[3][: d // 2]); rows.append(np.concatenate([h, -h]))      # symmetric: exact L/R ties
    rows.append(g.integers(-300, 301, d).astype(np.float32))                 # integers
    rows.append((g.integers(0, 3001, d) / 2.0).astype(np.float32))           # half-integers of the b=200 grid
    rows.append((g.integers(0, 201, d) * 0.125).astype(np.float32))          # dyadic grid
    rows.append(np.repeat(g.normal(size=16).astype(np.float32), d // 16))    # 16 repeated values
    r9 = g.normal(size=d).astype(np.float32) * 1e-3; r9[0] = -1.0; r9[1] = 1.0; rows.append(r9)   # one crowded bin
    r10 = g.normal(size=d).astype(np.float32); r10[7] = 40.0; rows.append(r10)                      # one outlier
    rows.append(np.linspace(-1, 1, d, dtype=np.float32))                     # uniform ramp
    rows.append((g.random(d) < 0.5).astype(np.float32) * 2 - 1)              # two values
    rows.append(g.standard_cauchy(d).astype(np.float32))                     # heavy tails
    rows.append((g.normal(size=d) * 1e-30).astype(np.float32))               # tiny magnitudes
    rows.append((g.normal(size=d) * 1e30).astype(np.float32))                # huge magnitudes
    x = np.ascontiguousarray(np.stack(rows).astype(np.float32))
    _, _, diag = _check(x, min_d=16)
    assert diag["deferred_rows"] >= 4, diag
    _check(x, "fp32", b=64, r=0.5, min_d=16)


def test_table_walk_nonfinite_row_reported():
    import paper_1911_02079_b200 as eq

    x = rng.mixed_table(64, 1024, 4)
    x[17, 500] = np.nan
    with pytest.raises(ValueError):
        eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "greedy", "fp16", 200, 0.16)


@pytest.mark.parametrize("at", [0, 1, 5, 7, 8, 9, 12, 15, 16, 17, 23, 24, 29, 31])
def test_table_walk_hand_over_at_every_iteration(at):
    """The walk settles six iterations per round and records its checkpoint (iteration 8k) from
    inside a round: hand every row over to the exact kernel at iteration `at` (development
    switch) -- restart list below iteration 8, resume records above -- and compare with the
    oracle.  Exercises the checkpoint taken at every position of a round."""
    x = rng.mixed_table(512, 1024, 1000 + at)
    os.environ["EQ4_DEV_TABLE_DEFER_AT"] = str(at)
    try:
        _, _, diag = _check(x, "fp16", min_d=16)
    finally:
        os.environ.pop("EQ4_DEV_TABLE_DEFER_AT", None)
    assert diag["deferred_rows"] == 512, diag
