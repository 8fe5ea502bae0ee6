"""Rows wider than the fused kernels' register/shared-memory sweet spot (d > 2048) and the other
parameters the reference accepts without limit (clipping.py:142-193, histclip.py:136-221,
codebook.py:35-138): bit-exact against the oracle."""

import numpy as np
import pytest
import torch

import oracle
import paper_1911_02079_b200 as eq
from oracle import rng
from test_oracle_golden import _bits

pytestmark = pytest.mark.gpu


def _check(x, method, aux, b=200, r=0.16, xd=None):
    p, rr = eq.quantize_pack_table4(torch.from_numpy(x).cuda() if xd is None else xd, method, aux, b, r,
                                    with_rows=True)
    want = oracle.quantize_pack_table(x, method, b, r, aux)
    st = eq.packed_row_stride(x.shape[1], aux)
    bad = np.nonzero((p.buffer.reshape(-1, st) != want.packed.reshape(-1, st)).any(1))[0]
    assert bad.size == 0, (method, x.shape, aux, bad[:8])
    assert np.array_equal(_bits(rr.xmin.cpu().numpy()), _bits(want.xmin))
    assert np.array_equal(_bits(rr.xmax.cpu().numpy()), _bits(want.xmax))
    return rr, want


@pytest.mark.parametrize("d", [2049, 3000, 4096, 4099, 6000, 8192, 12345, 16384])
def test_greedy_wide_rows(d):
    rows = max(4, 200_000 // d)
    x = rng.mixed_table(rows, d, d) if d % 2 else rng.sample_table("gaussian", 0.0, 1.0, d, rows, d)
    aux = "fp16" if d % 3 else "fp32"
    rr, want = _check(x, "greedy", aux)
    assert np.array_equal(rr.info0.cpu().numpy(), want.info0)


def test_greedy_wide_strided_view():
    """A wide table seen through a row pitch larger than d (masked kernels, unaligned rows)."""
    base = rng.sample_table("gaussian", 0.0, 1.0, 3, 24, 4200)
    xd = torch.from_numpy(base).cuda()[:, 3:3 + 4100]
    _check(np.ascontiguousarray(base[:, 3:3 + 4100]), "greedy", "fp16", xd=xd)


@pytest.mark.parametrize("method", ["asym", "sym", "table", "aciq", "gss"])
@pytest.mark.parametrize("d", [2049, 4096, 5001, 9000])
def test_rowwise_methods_wide_rows(method, d):
    rows = 48 if method != "gss" else 12
    x = rng.mixed_table(rows, d, d + 7)
    _check(x, method, "fp16" if d % 2 else "fp32")


@pytest.mark.parametrize("method,b,d", [("hist-brute", 200, 5000), ("hist-brute", 64, 20000),
                                        ("hist-apprx", 200, 12000), ("hist-brute", 4500, 64),
                                        ("hist-apprx", 5000, 64)])
def test_hist_wide_rows_and_many_bins(method, b, d):
    """Rows too wide to stage in shared memory (read from global memory) and b beyond the
    round-1 limits (4096 brute / 256 apprx): windows as the oracle's (norm ties excused)."""
    rows = (1 if method == "hist-brute" else 6) if b > 1000 else 24   # the oracle's scan is O(b^3)
    x = rng.mixed_table(rows, d, b + d)
    p, rr = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), method, "fp16", b, with_rows=True)
    st, ns = rr.info0.cpu().numpy(), rr.info1.cpu().numpy()
    for i, row in enumerate(x):
        if method == "hist-brute":
            o = oracle.hist_brute_search(row, b)
            if (st[i], ns[i]) != (o.start_bin, o.nbins_selected):
                ng = oracle.hist_window_norm(row, b, int(st[i]), int(ns[i]))
                assert abs(ng - o.norm) <= 1e-12 * abs(o.norm), (i, ng, o.norm)
        else:
            o, gap = oracle.hist_apprx_gap(row, b)
            if (st[i], ns[i]) != (o.start_bin, o.nbins_selected):
                assert gap <= 1e-12, i


@pytest.mark.parametrize("b,r", [(70000, 0.001), (100000, 0.0004)])
def test_greedy_many_bins(b, r):
    """b beyond 16 bits (round 1 refused b > 65535): a walk of ~b*r steps on the fine grid."""
    x = rng.mixed_table(64, 32, b)
    rr, want = _check(x, "greedy", "fp16", b=b, r=r)
    assert np.array_equal(rr.info0.cpu().numpy(), want.info0)
