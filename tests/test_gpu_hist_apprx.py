"""GPU HIST-APPRX (histclip.py:181-217) against the reference's windows (tests/golden/
hist_apprx.npz) and the oracle.  The reference's window norms go through numpy's SIMD pow
(host-dependent in the last bit), so windows must be identical except where the walk met a
near-tie (|nl - nr| <= 1e-12 relative, checked with the oracle); norms agree to 1e-12."""

import numpy as np
import pytest
import torch

import oracle
import paper_1911_02079_b200 as eq
from oracle import rng
from test_oracle_golden import _load

pytestmark = pytest.mark.gpu
TIE = 1e-12


def _check(x, b, st, ns, lo, hi):
    p, rr = eq.quantize_pack_table4(torch.from_numpy(np.ascontiguousarray(x)).cuda(), "hist-apprx",
                                    "fp16", b, with_rows=True)
    gst, gns = rr.info0.cpu().numpy(), rr.info1.cpu().numpy()
    glo, ghi, gnorm = rr.xmin.cpu().numpy(), rr.xmax.cpu().numpy(), rr.norm.cpu().numpy()
    ties = 0
    for i in range(x.shape[0]):
        if (gst[i], gns[i]) != (st[i], ns[i]):
            _, gap = oracle.hist_apprx_gap(x[i], b)
            assert gap <= TIE, (i, gap)
            ties += 1
            continue
        assert (glo[i], ghi[i]) == (lo[i], hi[i]), i
        o = oracle.hist_apprx_search(x[i], b)
        assert abs(gnorm[i] - o.norm) <= 1e-12 * max(1.0, abs(o.norm)), i
    return p, ties


def test_hist_apprx_reference_windows():
    f = _load("hist_apprx.npz")
    for tname in ("gauss64", "lap64", "mixed33"):
        x = f[f"x_{tname}"]
        for b in (200, 40, 8):
            st, ns = f[f"win_{tname}_{b}"]
            lo, hi = f[f"range_{tname}_{b}"]
            p, ties = _check(x, b, st, ns, lo, hi)
            assert ties == 0, (tname, b)
            if b == 200:
                assert np.array_equal(p.buffer, f[f"packed_{tname}"]), tname


@pytest.mark.parametrize("rows,d,b", [(3000, 64, 200), (1000, 17, 256), (2000, 128, 100), (500, 300, 200),
                                      (300, 64, 1), (300, 9, 2), (200, 2048, 64), (400, 1, 16)])
def test_hist_apprx_vs_oracle(rows, d, b):
    x = rng.mixed_table(rows, d, d + b)
    want = oracle.quantize_pack_table(x, "hist-apprx", b, 0.16, "fp16")
    p, ties = _check(x, b, want.info0, want.info1, want.xmin, want.xmax)
    assert ties <= rows // 1000
    if ties == 0:
        assert np.array_equal(p.buffer, want.packed)


def test_hist_apprx_api_and_counters():
    x = rng.sample_table("gaussian", 0.0, 1.0, 9, 4, 64)
    for row in x:
        c = eq.WorkCounters()
        h = eq.hist_apprx_search(row, 200, counters=c)
        o = oracle.hist_apprx_search(row, 200)
        assert (h.start_bin, h.nbins_selected) == (o.start_bin, o.nbins_selected)
        assert (c.candidate_evals, c.bin_visits) == (o.candidate_evals, o.bin_visits)
    c = eq.WorkCounters()
    eq.row_clip_range("hist-apprx", np.full(9, 2.5, np.float32), b=40, counters=c)
    assert (c.candidate_evals, c.bin_visits) == (1, 40)
    h = eq.hist_apprx_search(x[0], 300)          # b > 256: numpy leaves beyond two
    o = oracle.hist_apprx_search(x[0], 300)
    assert (h.start_bin, h.nbins_selected) == (o.start_bin, o.nbins_selected)


@pytest.mark.parametrize("b", [249, 250, 253, 255, 257, 300, 400, 1000])
def test_hist_apprx_pairwise_leaves(b):
    """b in 249..255 (the right half of 129..135 terms splits again), and b > 256: windows
    identical to the oracle's except where its walk meets a 1e-12 near-tie, norms within
    1e-12."""
    x = rng.mixed_table(300, 64, b)
    p, rr = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "hist-apprx", "fp16", b, with_rows=True)
    st, ns, nm = rr.info0.cpu().numpy(), rr.info1.cpu().numpy(), rr.norm.cpu().numpy()
    for i, row in enumerate(x):
        o, gap = oracle.hist_apprx_gap(row, b)
        if (st[i], ns[i]) != (o.start_bin, o.nbins_selected):
            assert gap <= 1e-12, (b, i)
            continue
        assert nm[i] == pytest.approx(o.norm, rel=1e-12, abs=1e-300), (b, i)
