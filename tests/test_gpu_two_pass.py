"""GREEDY two-pass scheme (vector rows): the fp32 screening kernel k_greedy_fast defers the rows
whose walk meets a comparison inside the error band (and rows it does not take: zero min/max,
constant, non-finite, coarse reference grid) to k_greedy in list mode.  The bytes, float64
ranges, iteration counts and best pairs must equal both the oracle's and the single-kernel
path's (k_greedy over every row, selected with the development switch EQ4_DEV_ONE_PASS)."""

import os

import numpy as np
import pytest

import oracle
from oracle import rng

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _run(eq, x, one_pass, env=None):
    if one_pass:
        os.environ["EQ4_DEV_ONE_PASS"] = "1"
    for k, v in (env or {}).items():
        os.environ[k] = v
    try:
        rows, d = x.shape
        out = torch.zeros(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
        rr = eq.RowResults(torch.zeros(rows, dtype=torch.float64, device="cuda"),
                           torch.zeros(rows, dtype=torch.float64, device="cuda"),
                           torch.full((rows,), -7, dtype=torch.int32, device="cuda"),
                           torch.full((rows,), -7, dtype=torch.int32, device="cuda"), None)
        from paper_1911_02079_b200 import _lib
        _lib.diag_counters(reset=True)
        eq.quantize_pack_table4(x, "greedy", "fp16", 200, 0.16, out=out, rows_out=rr)
        torch.cuda.synchronize()
        diag = _lib.diag_counters(reset=True)
        return out.cpu().numpy(), rr, diag
    finally:
        os.environ.pop("EQ4_DEV_ONE_PASS", None)
        for k in (env or {}):
            os.environ.pop(k, None)


@pytest.mark.parametrize("d,rows", [(16, 40_000), (64, 30_000), (128, 12_000), (1024, 1_500)])
def test_two_pass_matches_one_pass_and_oracle(d, rows):
    import paper_1911_02079_b200 as eq

    xh = rng.mixed_table(rows, d, 7 + d)
    # rows the screen must hand over: a zero minimum, a zero maximum, a constant row,
    # a row with a huge offset (coarse reference grid)
    xh[5, :] = np.abs(xh[5, :]); xh[5, 3] = 0.0
    xh[6, :] = -np.abs(xh[6, :]); xh[6, 1] = 0.0
    xh[7, :] = 1.25
    xh[8, :] = xh[8, :] * 1e-9 + 3e4
    x = torch.from_numpy(xh).cuda()
    got, rr, diag = _run(eq, x, one_pass=False)
    ref, rr1, _ = _run(eq, x, one_pass=True)
    assert diag["deferred_rows"] >= 4, diag          # the four crafted rows at least
    assert np.array_equal(got, ref)
    for f in ("xmin", "xmax", "info0", "info1"):
        assert torch.equal(getattr(rr, f), getattr(rr1, f)), f
    want = oracle.quantize_pack_table(xh, "greedy", 200, 0.16, "fp16")
    assert np.array_equal(got, want.packed)
    assert np.array_equal(rr.xmin.cpu().numpy(), want.xmin)
    assert np.array_equal(rr.xmax.cpu().numpy(), want.xmax)
    assert np.array_equal(rr.info0.cpu().numpy(), want.info0)


def test_two_pass_all_rows_deferred():
    """Every row handed over (all constant): the list holds the whole table."""
    import paper_1911_02079_b200 as eq

    xh = np.repeat(np.linspace(-1, 1, 3000, dtype=np.float32)[:, None], 64, axis=1)
    x = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    got, rr, diag = _run(eq, x, one_pass=False)
    assert diag["deferred_rows"] == 3000
    want = oracle.quantize_pack_table(xh, "greedy", 200, 0.16, "fp16")
    assert np.array_equal(got, want.packed)


@pytest.mark.parametrize("env", [{"EQ4_DEV_RCAP": "40"}, {"EQ4_DEV_NO_RESUME": "1"}])
def test_two_pass_resume_overflow_and_restart(env):
    """Deferred rows resume from the screen's last checkpoint (iteration 8k) when their group has
    room and restart otherwise: a 40-record cap (most resumable rows overflow to the restart list)
    and resuming switched off give the same bytes as the one-kernel path."""
    import paper_1911_02079_b200 as eq

    xh = rng.mixed_table(20_000, 64, 31)
    x = torch.from_numpy(xh).cuda()
    got, rr, diag = _run(eq, x, one_pass=False, env=env)
    ref, rr1, _ = _run(eq, x, one_pass=True)
    assert diag["deferred_rows"] > 100, diag
    assert np.array_equal(got, ref)
    for f in ("xmin", "xmax", "info0", "info1"):
        assert torch.equal(getattr(rr, f), getattr(rr1, f)), f
