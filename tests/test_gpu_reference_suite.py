"""The reference package's own hot-path tests, restated against the B200 drop-in.

Each test below restates one test of /root/reference/pkg/tests (same class and test
names, same inputs and assertions; SURVEY.md section 4 lists the hot-path files) with the
reference's names bound to ``paper_1911_02079_b200`` -- so every value asserted here is
computed by libeq4.so on the GPU:
  test_table.py    11-80   (containers, quant_mse)
  test_codec.py    17-110  (quantize_uniform / dequantize_uniform, round-trip bound)
  test_clipping.py 28-211  (sym/asym/table/gss/aciq/greedy ranges, equivariance)
  test_histclip.py 22-138  (build_histogram, bin_l2_norm, hist-brute, hist-apprx)
  test_packed.py   39-100  (packing layout, unpack_row)
The reference's scalar test oracles (pkg/tests/oracles.py) are replaced by this repo's C
oracle (oracle/, pinned to the reference by tests/test_oracle_golden.py) and two short
scalar helpers restated below; gaussian_row / laplacian_row come from the pinned numpy
port of the reference's generator (oracle/rng.py).
"""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
import paper_1911_02079_b200 as embquant
from oracle import rng
from paper_1911_02079_b200 import (ClipRange, EmbeddingTable, UniformQuantTable, WorkCounters,
                                   bin_l2_norm, build_histogram, clip_range_aciq, clip_range_asym,
                                   clip_range_greedy, clip_range_gss, clip_range_hist_apprx,
                                   clip_range_hist_brute, clip_range_sym, clip_range_table,
                                   dequantize_uniform, hist_apprx_search, hist_brute_search,
                                   pack_table4, quant_mse, quantize_table, quantize_table_uniform,
                                   quantize_uniform, unpack_row, unpack_row_codes)

pytestmark = pytest.mark.gpu


def gaussian_row(seed, d, mean=0.0, std=1.0):
    """oracles.py:18-19: sample_table(RngSpec("gaussian", mean, std, seed), 1, d).row(0)."""
    return rng.sample_table("gaussian", mean, std, seed, 1, d)[0]


def laplacian_row(seed, d, loc=0.0, scale=1.0):
    """oracles.py:22-23."""
    return rng.sample_table("laplacian", loc, scale, seed, 1, d)[0]


def scalar_quant_mse(x, xmin, xmax, nbits):
    """oracles.py:26-42, restated: straight-line scalar codec error."""
    total = 0.0
    if xmax == xmin:
        return sum((float(v) - xmin) ** 2 for v in x)
    qmax = (1 << nbits) - 1
    scale = (xmax - xmin) / qmax
    for v in x:
        v = float(v)
        code = min(max(math.floor((min(max(v, xmin), xmax) - xmin) / scale + 0.5), 0), qmax)
        total += (v - (scale * code + xmin)) ** 2
    return total


def scalar_histogram(x, b):
    """oracles.py:45-58, restated: (lo, hi, counts), half-open bins, last bin closed."""
    lo, hi = float(min(x)), float(max(x))
    counts = [0] * b
    if lo == hi:
        counts[0] = len(x)
        return lo, hi, counts
    w = (hi - lo) / b
    for v in x:
        counts[min(max(int(math.floor((float(v) - lo) / w)), 0), b - 1)] += 1
    return lo, hi, counts


def brute_best_window(x, b):
    """oracles.py:99-112 via the C oracle's literal window scan: ((start, n), norm)."""
    h = oracle.hist_brute_search(np.asarray(x, np.float32), b)
    return (h.start_bin, h.nbins_selected), h.norm


def table_normalized_l2(t, recon):
    """metrics.py:47-62 flattened mode (test helper only: quality metrics are outside the
    hot path): sqrt(sum sq err) / sqrt(sum sq)."""
    t = np.asarray(t.values if isinstance(t, EmbeddingTable) else t, np.float64).ravel()
    r = np.asarray(recon, np.float64).ravel()
    return float(np.linalg.norm(t - r) / np.linalg.norm(t))


# ---------------------------------------------------------------------------
# test_table.py
# ---------------------------------------------------------------------------
class TestEmbeddingTable:
    def test_row_layout(self):
        t = EmbeddingTable(np.array([[1, 2, 3], [4, 5, 6]], dtype=np.float32))
        assert t.row(0).tolist() == [1, 2, 3]
        assert t.row(1).tolist() == [4, 5, 6]

    def test_row_out_of_bounds(self):
        t = EmbeddingTable(np.ones((2, 3), dtype=np.float32))
        with pytest.raises(IndexError):
            t.row(2)
        with pytest.raises(IndexError):
            t.row(-1)

    def test_rejects_non_finite(self):
        with pytest.raises(ValueError):
            EmbeddingTable(np.array([[1.0, np.nan]], dtype=np.float32))
        with pytest.raises(ValueError):
            EmbeddingTable(np.array([[np.inf, 1.0]], dtype=np.float32))

    def test_rejects_empty(self):
        with pytest.raises(ValueError):
            EmbeddingTable(np.zeros((0, 4), dtype=np.float32))

    def test_values_read_only(self):
        t = EmbeddingTable(np.ones((2, 2), dtype=np.float32))
        with pytest.raises(ValueError):
            t.values[0, 0] = 5.0


class TestClipRange:
    def test_orders_endpoints(self):
        with pytest.raises(ValueError):
            ClipRange(1.0, -1.0)

    def test_rejects_non_finite(self):
        with pytest.raises(ValueError):
            ClipRange(0.0, np.inf)


class TestQuantMse:
    def test_exact_grid_is_zero(self):
        x = np.arange(16, dtype=np.float64)
        assert quant_mse(x, ClipRange(0.0, 15.0), 4) == 0.0

    def test_half_grid_point(self):
        assert quant_mse([0.5], ClipRange(0.0, 15.0), 4) == pytest.approx(0.25, abs=0)

    def test_matches_scalar_reference(self):
        x = gaussian_row(7, 64)
        r = ClipRange(float(x.min()), float(x.max()))
        assert quant_mse(x, r, 4) == pytest.approx(scalar_quant_mse(x, r.xmin, r.xmax, 4), rel=1e-12)

    def test_degenerate_range(self):
        assert quant_mse([2.5, 2.5], ClipRange(2.5, 2.5), 4) == 0.0
        assert quant_mse([3.5], ClipRange(2.5, 2.5), 4) == pytest.approx(1.0)

    @given(st.lists(st.floats(-50, 50), min_size=1, max_size=40), st.randoms())
    @settings(max_examples=60, deadline=None)
    def test_permutation_invariant_and_nonnegative(self, values, rnd):
        x = np.array(values)
        r = ClipRange(float(x.min()) - 0.5, float(x.max()) + 1.0)
        base = quant_mse(x, r, 4)
        assert base >= 0.0
        shuffled = list(values)
        rnd.shuffle(shuffled)
        assert quant_mse(np.array(shuffled), r, 4) == pytest.approx(base, rel=1e-12, abs=1e-12)
        # and bit-exact against the oracle's numpy restatement (float64 values)
        assert base == _oracle_quant_mse_f64(x, r)


def _oracle_quant_mse_f64(x, r):
    """table.py:81-103 in numpy float64 with the oracle's pairwise sum (test helper)."""
    x = np.asarray(x, np.float64)
    if r.xmax == r.xmin:
        return oracle.np_sum((x - r.xmin) ** 2)
    scale = (r.xmax - r.xmin) / 15
    codes = np.clip(np.floor((np.clip(x, r.xmin, r.xmax) - r.xmin) / scale + 0.5), 0, 15)
    return oracle.np_sum((x - (scale * codes + r.xmin)) ** 2)


# ---------------------------------------------------------------------------
# test_codec.py
# ---------------------------------------------------------------------------
class TestQuantizeUniform:
    def test_exact_grid(self):
        q = quantize_uniform(np.arange(16.0), ClipRange(0.0, 15.0), 4)
        assert float(q.scale) == 1.0
        assert float(q.bias) == 0.0
        assert q.codes.tolist() == list(range(16))

    def test_endpoints_map_to_extreme_codes(self):
        q = quantize_uniform([-1.0, 1.0], ClipRange(-1.0, 1.0), 4)
        assert q.codes.tolist() == [0, 15]
        assert float(q.scale) == pytest.approx(2.0 / 15.0)
        assert float(q.bias) == -1.0

    def test_clamp_and_tie_rounding(self):
        q = quantize_uniform([100.0, 0.0, -3.0], ClipRange(-3.0, 3.0), 4)
        assert q.codes.tolist() == [15, 8, 0]

    def test_constant_row_convention(self):
        q = quantize_uniform([2.5, 2.5], ClipRange(2.5, 2.5), 4)
        assert float(q.scale) == 0.0
        assert q.codes.tolist() == [0, 0]
        assert dequantize_uniform(q).tolist() == [2.5, 2.5]

    def test_8bit_codes(self):
        q = quantize_uniform(np.linspace(0, 255, 256), ClipRange(0.0, 255.0), 8)
        assert q.codes.tolist() == list(range(256))

    def test_rejects_bad_nbits(self):
        with pytest.raises(ValueError):
            quantize_uniform([1.0], ClipRange(0.0, 1.0), 5)


class TestDequantizeUniform:
    def test_identity_grid(self):
        q = quantize_uniform(np.arange(16.0), ClipRange(0.0, 15.0), 4)
        assert dequantize_uniform(q).tolist() == [float(i) for i in range(16)]

    def test_endpoint_reconstruction(self):
        q = quantize_uniform([-1.0, 1.0], ClipRange(-1.0, 1.0), 4)
        deq = dequantize_uniform(q)
        ulp = np.spacing(np.float32(1.0))
        assert abs(deq[0] - (-1.0)) <= ulp
        assert abs(deq[1] - 1.0) <= ulp

    def test_float32_output(self):
        q = quantize_uniform([0.3, 0.7], ClipRange(0.0, 1.0), 4)
        assert dequantize_uniform(q).dtype == np.float32

    def test_fp16_aux_widened(self):
        x = gaussian_row(21, 32)
        r = ClipRange(float(x.min()), float(x.max()))
        q32 = quantize_uniform(x, r, 4, "fp32")
        q16 = quantize_uniform(x, r, 4, "fp16")
        assert q16.scale.dtype == np.float16
        assert np.array_equal(q32.codes, q16.codes)
        assert np.allclose(dequantize_uniform(q32), dequantize_uniform(q16), rtol=2e-3, atol=2e-3)


def _roundtrip_bound(x, xmin, xmax, nbits):
    """test_codec.py:82-90: |x - deq(quant(x))| <= scale/2 + 4 ulp for in-range values."""
    q = quantize_uniform(x, ClipRange(xmin, xmax), nbits)
    deq = dequantize_uniform(q).astype(np.float64)
    scale = (xmax - xmin) / ((1 << nbits) - 1)
    err = np.abs(np.asarray(x, dtype=np.float64) - deq)
    ulp = np.spacing(np.maximum(np.abs(x), np.abs(deq)).astype(np.float32)).astype(np.float64)
    return err, scale / 2.0 + 4.0 * ulp


class TestRoundTripBound:
    @given(st.floats(-1e4, 1e4), st.floats(1e-6, 1e4), st.integers(0, 100), st.sampled_from([4, 8]))
    @settings(max_examples=200, deadline=None)
    def test_in_range_values(self, xmin, width, pick, nbits):
        xmax = xmin + width
        x = np.float32(xmin + width * pick / 100.0)
        err, bound = _roundtrip_bound(np.array([x]), xmin, xmax, nbits)
        assert err[0] <= bound[0]

    def test_gaussian_rows(self):
        for seed in range(20):
            x = gaussian_row(seed, 64)
            err, bound = _roundtrip_bound(x, float(x.min()), float(x.max()), 4)
            assert np.all(err <= bound)


# ---------------------------------------------------------------------------
# test_clipping.py
# ---------------------------------------------------------------------------
def _table(seed, rows, dim):
    return EmbeddingTable(np.stack([gaussian_row(seed * 1000 + i, dim) for i in range(rows)]))


class TestSymAsym:
    def test_sym_examples(self):
        assert clip_range_sym([-3.0, 1.0]) == ClipRange(-3.0, 3.0)
        assert clip_range_sym([0.0, 0.0]) == ClipRange(0.0, 0.0)
        assert clip_range_sym([5.0]) == ClipRange(-5.0, 5.0)

    def test_sym_exact_negation(self):
        r = clip_range_sym(gaussian_row(3, 33))
        assert r.xmin == -r.xmax

    def test_asym_examples(self):
        assert clip_range_asym([-3.0, 1.0]) == ClipRange(-3.0, 1.0)
        assert clip_range_asym([7.0]) == ClipRange(7.0, 7.0)
        assert clip_range_asym([1.0, 2.0, 100.0]) == ClipRange(1.0, 100.0)

    def test_empty_rejected(self):
        with pytest.raises(ValueError):
            clip_range_sym([])
        with pytest.raises(ValueError):
            clip_range_asym([])


class TestTableRange:
    def test_min_max_over_all(self):
        t = EmbeddingTable(np.array([[0.0, 1.0], [-2.0, 3.0]], dtype=np.float32))
        assert clip_range_table(t) == ClipRange(-2.0, 3.0)

    def test_single_row_equals_asym(self):
        t = _table(4, 1, 16)
        assert clip_range_table(t) == clip_range_asym(t.row(0))

    def test_rowwise_asym_beats_table_in_aggregate(self):
        t = _table(11, 10, 64)
        la = table_normalized_l2(t, quantize_table(t, "asym").dequantize())
        lt = table_normalized_l2(t, quantize_table(t, "table").dequantize())
        assert la <= lt


class TestGss:
    def test_two_point_symmetric(self):
        r = clip_range_gss([-1.0, 1.0])
        assert r.xmax == pytest.approx(1.0, rel=1e-9)
        assert r.xmin == -r.xmax

    def test_beats_clipping_at_fixed_threshold(self):
        # float64 values float32 cannot hold: the GSS search runs on the float64 row
        x = np.concatenate([np.arange(-15, 16) / 15.0, [8.0, -8.0]])
        r = clip_range_gss(x)
        loss = quant_mse(x, r, 4)
        grid = np.linspace(1e-3, float(np.max(np.abs(x))), 10**4)
        assert loss <= min(quant_mse(x, ClipRange(-t, t), 4) for t in [8.0])
        dense_best = min(quant_mse(x, ClipRange(-t, t), 4) for t in grid)
        assert loss <= dense_best * 1.05

    def test_never_loses_to_sym(self):
        for seed in range(30):
            x = gaussian_row(seed + 50, 64)
            assert quant_mse(x, clip_range_gss(x), 4) <= quant_mse(x, clip_range_sym(x), 4)

    def test_all_zero(self):
        assert clip_range_gss([0.0, 0.0, 0.0]) == ClipRange(0.0, 0.0)


class TestAciq:
    def test_formula_on_two_points(self):
        r = clip_range_aciq([-1.0, 1.0], "laplacian")
        assert r.xmin == pytest.approx(-5.03)
        assert r.xmax == pytest.approx(5.03)

    def test_constant_falls_back(self):
        assert clip_range_aciq([3.0, 3.0, 3.0]) == ClipRange(3.0, 3.0)

    def test_matches_recomputed_mad(self):
        x = laplacian_row(9, 128)
        r = clip_range_aciq(x)
        mu = float(np.mean(np.asarray(x, dtype=np.float64)))
        mad = float(np.mean(np.abs(np.asarray(x, dtype=np.float64) - mu)))
        assert r.xmin == pytest.approx(mu - 5.03 * mad, rel=1e-12)
        assert r.xmax == pytest.approx(mu + 5.03 * mad, rel=1e-12)

    def test_gaussian_requires_constant(self):
        with pytest.raises(ValueError):
            clip_range_aciq([1.0, 2.0], "gaussian")
        r = clip_range_aciq([-1.0, 1.0], "gaussian", gaussian_constant=2.0)
        assert r.xmax == pytest.approx(2.0)


class TestGreedy:
    def test_exact_grid_keeps_full_range(self):
        x = np.arange(16.0)
        r = clip_range_greedy(x, 4)
        assert r == ClipRange(0.0, 15.0)
        assert quant_mse(x, r, 4) == 0.0

    def test_outlier_forces_clipping_win(self):
        x = np.concatenate([gaussian_row(13, 63), np.float32([100.0])])
        assert quant_mse(x, clip_range_greedy(x, 4), 4) < quant_mse(x, clip_range_asym(x), 4)

    def test_never_loses_to_asym(self):
        for seed in range(50):
            x = gaussian_row(seed + 200, 32)
            assert quant_mse(x, clip_range_greedy(x, 4), 4) <= quant_mse(x, clip_range_asym(x), 4)

    def test_constant_input(self):
        assert clip_range_greedy([4.0, 4.0], 4) == ClipRange(4.0, 4.0)

    def test_evaluation_count(self):
        counters = WorkCounters()
        clip_range_greedy(gaussian_row(5, 64), 4, 200, 0.16, counters=counters)
        assert abs(counters.loss_evals - 2 * 200 * 0.16) <= 200

    def test_budget_tradeoff_against_stock(self):
        stock_losses, opt_losses = [], []
        for seed in range(100):
            x = gaussian_row(5000 + seed, 64)
            asym = quant_mse(x, clip_range_asym(x), 4)
            stock = quant_mse(x, clip_range_greedy(x, 4, 200, 0.16), 4)
            opt = quant_mse(x, clip_range_greedy(x, 4, 1000, 0.5), 4)
            assert stock <= asym and opt <= asym
            stock_losses.append(stock)
            opt_losses.append(opt)
        assert np.mean(opt_losses) <= np.mean(stock_losses) * 1.02
        assert np.mean(stock_losses) <= np.mean(opt_losses) * 1.02

    def test_rejects_bad_params(self):
        with pytest.raises(ValueError):
            clip_range_greedy([1.0, 2.0], 4, b=0)
        with pytest.raises(ValueError):
            clip_range_greedy([1.0, 2.0], 4, r=0.0)


class TestEquivariance:
    METHODS = {"sym": clip_range_sym, "asym": clip_range_asym, "gss": clip_range_gss,
               "aciq": clip_range_aciq, "greedy": clip_range_greedy}

    def test_negation_maps_asym_range(self):
        x = gaussian_row(31, 48)
        r = clip_range_asym(x)
        assert clip_range_asym(-x) == ClipRange(-r.xmax, -r.xmin)

    def test_negation_fixes_sym_and_losses(self):
        x = gaussian_row(32, 48)
        assert clip_range_sym(-x) == clip_range_sym(x)
        for name in ("sym", "gss"):
            r, rn = self.METHODS[name](x), self.METHODS[name](-x)
            assert quant_mse(x, r, 4) == pytest.approx(quant_mse(-x, rn, 4), rel=1e-12)

    @pytest.mark.parametrize("c", [0.25, 4.0, 1024.0])
    def test_power_of_two_scaling_is_exact(self, c):
        x = gaussian_row(33, 48)
        xs = (x.astype(np.float64) * c).astype(np.float32)
        for name, fn in self.METHODS.items():
            r, rs = fn(x), fn(xs)
            if r.xmax != r.xmin:
                assert rs.xmin == pytest.approx(c * r.xmin, rel=1e-6)
                assert rs.xmax == pytest.approx(c * r.xmax, rel=1e-6)
            nb = np.sqrt(quant_mse(x, r, 4)) / np.linalg.norm(x.astype(np.float64))
            ns = np.sqrt(quant_mse(xs, rs, 4)) / np.linalg.norm(xs.astype(np.float64))
            assert ns == pytest.approx(nb, rel=1e-9, abs=1e-12)


# ---------------------------------------------------------------------------
# test_histclip.py
# ---------------------------------------------------------------------------
class TestBuildHistogram:
    def test_two_bins(self):
        assert build_histogram([0.0, 1.0], 2).counts.tolist() == [1, 1]

    def test_half_open_bins(self):
        assert build_histogram([0.0, 0.49, 0.51, 1.0], 2).counts.tolist() == [2, 2]

    def test_degenerate_constant(self):
        h = build_histogram([5.0, 5.0, 5.0], 4)
        assert h.counts.tolist() == [3, 0, 0, 0]
        assert h.lo == h.hi == 5.0

    def test_mass_conserved_and_matches_scalar(self):
        for seed in range(10):
            x = gaussian_row(seed, 64)
            h = build_histogram(x, 20)
            assert int(h.counts.sum()) == 64
            assert h.counts.tolist() == scalar_histogram(x, 20)[2]


class TestBinL2Norm:
    def test_symmetric_interval(self):
        w, rho = 0.8, 3.0
        assert bin_l2_norm(-w / 2, w / 2, rho) == pytest.approx(rho * w ** 3 / 12)

    def test_empty_interval(self):
        assert bin_l2_norm(0.0, 0.0, 7.0) == 0.0

    def test_unit_case(self):
        assert bin_l2_norm(0.0, 1.0, 3.0) == pytest.approx(1.0)

    def test_arrays_broadcast(self):
        db, de = np.array([-0.5, 0.0, 1.0]), np.array([0.5, 2.0, 1.0])
        want = 2.0 * (de ** 3 - db ** 3) / 3.0
        np.testing.assert_allclose(bin_l2_norm(db, de, 2.0), want, rtol=1e-15)


class TestHistBrute:
    def test_constant_input(self):
        assert clip_range_hist_brute([4.0, 4.0, 4.0], 16) == ClipRange(4.0, 4.0)

    @pytest.mark.parametrize("b", [8, 16, 40])
    def test_selection_matches_literal_rescan(self, b):
        for seed in range(5):
            x = gaussian_row(seed * 31 + 1, 64)
            got = hist_brute_search(x, b)
            (want_start, want_n), want_norm = brute_best_window(x, b)
            assert (got.start_bin, got.nbins_selected) == (want_start, want_n)
            assert got.norm == pytest.approx(want_norm, rel=1e-9)

    def test_outlier_prefix_selection(self):
        dense = rng.uniform_open01(123, 4000).astype(np.float32)
        x = np.concatenate([dense, np.float32([25.0])])
        b = 40
        got = hist_brute_search(x, b)
        (want_start, want_n), want_norm = brute_best_window(x, b)
        assert (got.start_bin, got.nbins_selected) == (want_start, want_n)
        assert got.start_bin == 0
        assert got.clip_range.xmax < 12.5

    def test_window_range_mapping(self):
        x = gaussian_row(8, 64)
        b = 16
        got = hist_brute_search(x, b)
        h = build_histogram(x, b)
        w = h.bin_width
        assert got.clip_range.xmin == pytest.approx(h.lo + w * got.start_bin)
        assert got.clip_range.xmax == pytest.approx(h.lo + w * (got.start_bin + got.nbins_selected))

    def test_counters_grow_cubically(self):
        x = gaussian_row(5, 64)
        c200, c400 = WorkCounters(), WorkCounters()
        clip_range_hist_brute(x, 200, counters=c200)
        clip_range_hist_brute(x, 400, counters=c400)
        assert 8.0 * 0.85 <= c400.bin_visits / c200.bin_visits <= 8.0 * 1.15
        assert 3.5 <= c400.candidate_evals / c200.candidate_evals <= 4.5


class TestHistApprx:
    def test_full_grid_retained(self):
        assert clip_range_hist_apprx(np.arange(16.0), 16) == ClipRange(0.0, 15.0)

    def test_constant_input(self):
        assert clip_range_hist_apprx([2.0, 2.0], 8) == ClipRange(2.0, 2.0)

    def test_linear_candidate_count(self):
        counters = WorkCounters()
        clip_range_hist_apprx(gaussian_row(6, 64), 200, counters=counters)
        assert counters.candidate_evals <= 2 * 200 + 1

    def test_never_beats_brute_norm_and_close_loss(self):
        rel_diffs = []
        for seed in range(60):
            x = gaussian_row(900 + seed, 64)
            brute, apprx = hist_brute_search(x, 200), hist_apprx_search(x, 200)
            assert apprx.norm >= brute.norm - 1e-12 * max(1.0, brute.norm)
            lb, la = quant_mse(x, brute.clip_range, 4), quant_mse(x, apprx.clip_range, 4)
            rel_diffs.append(abs(la - lb) / lb)
        assert float(np.mean(rel_diffs)) < 0.25

    def test_apprx_window_is_brute_candidate(self):
        x = gaussian_row(41, 64)
        b = 24
        apprx = hist_apprx_search(x, b)
        want = oracle.hist_window_norm(x, b, apprx.start_bin, apprx.nbins_selected)
        assert apprx.norm == pytest.approx(want, rel=1e-9)


# ---------------------------------------------------------------------------
# test_packed.py
# ---------------------------------------------------------------------------
def _qtable(codes, scale=1.0, bias=0.0, aux="fp32"):
    codes = np.atleast_2d(np.asarray(codes, dtype=np.uint8))
    n = codes.shape[0]
    return UniformQuantTable(codes, np.full(n, scale), np.full(n, bias), 4, aux)


def _random_packed(seed, rows, dim, aux="fp32"):
    t = EmbeddingTable(np.stack([gaussian_row(seed + i, dim) for i in range(rows)]))
    ranges = [clip_range_asym(t.row(i)) for i in range(rows)]
    return t, pack_table4(quantize_table_uniform(t, ranges, 4, aux))


class TestPacking:
    def test_nibble_order(self):
        assert pack_table4(_qtable([[1, 2]])).buffer[0] == 0x21

    def test_odd_d_pad(self):
        assert pack_table4(_qtable([[15]])).buffer[0] == 0x0F

    def test_rejects_8bit(self):
        q = UniformQuantTable(np.zeros((1, 4), dtype=np.uint8), [1.0], [0.0], 8)
        with pytest.raises(ValueError):
            pack_table4(q)

    def test_roundtrip_random_rows(self):
        r = np.random.default_rng(99)
        codes = r.integers(0, 16, size=(100, 7)).astype(np.uint8)
        scales = np.linspace(0.01, 2.0, 100).astype(np.float32)
        biases = np.linspace(-3.0, 3.0, 100).astype(np.float32)
        p = pack_table4(UniformQuantTable(codes, scales, biases, 4))
        for i in range(100):
            got_codes, got_scale, got_bias = unpack_row_codes(p, i)
            assert np.array_equal(got_codes, codes[i])
            assert got_scale == scales[i] and got_bias == biases[i]

    @given(st.lists(st.integers(0, 15), min_size=1, max_size=33))
    @settings(max_examples=80, deadline=None)
    def test_packing_bijection(self, code_list):
        got, _, _ = unpack_row_codes(pack_table4(_qtable([code_list])), 0)
        assert got.tolist() == code_list

    def test_row_stride(self):
        assert pack_table4(_qtable([[0] * 128])).row_stride == 64 + 8
        assert pack_table4(_qtable([[0] * 128], aux="fp16")).row_stride == 64 + 4
        assert pack_table4(_qtable([[0] * 7])).row_stride == 4 + 8


class TestUnpackRow:
    def test_known_bytes(self):
        assert unpack_row(pack_table4(_qtable([[1, 2]], scale=1.0, bias=0.0)), 0).tolist() == [1.0, 2.0]
        assert unpack_row(pack_table4(_qtable([[1, 2]], scale=0.5, bias=-1.0)), 0).tolist() == [-0.5, 0.0]

    def test_fp16_aux_identity_values(self):
        p32 = pack_table4(_qtable([[3, 9]], scale=1.0, bias=0.0, aux="fp32"))
        p16 = pack_table4(_qtable([[3, 9]], scale=1.0, bias=0.0, aux="fp16"))
        assert np.array_equal(unpack_row(p32, 0), unpack_row(p16, 0))

    def test_matches_dequantize(self):
        t, p = _random_packed(700, 10, 17)
        ranges = [clip_range_asym(t.row(i)) for i in range(10)]
        deq = quantize_table_uniform(t, ranges, 4).dequantize()
        for i in range(10):
            assert np.array_equal(unpack_row(p, i), deq[i])

    def test_bounds(self):
        _, p = _random_packed(800, 3, 5)
        with pytest.raises(IndexError):
            unpack_row(p, 3)


# ---------------------------------------------------------------------------
# the drop-in against the oracle on the same helpers (bit-exact)
# ---------------------------------------------------------------------------
def test_codec_and_histogram_vs_oracle():
    r = np.random.default_rng(5)
    x = rng.mixed_table(300, 37, 5)
    lo, hi = x.min(axis=1).astype(np.float64), x.max(axis=1).astype(np.float64)
    lo = lo + 0.1 * (hi - lo) * r.random(300)          # clipping ranges inside the data range
    ranges = [ClipRange(a, b) for a, b in zip(lo, hi)]
    for aux in ("fp16", "fp32"):
        q = quantize_table_uniform(EmbeddingTable(x), ranges, 4, aux)
        for i in range(0, 300, 7):
            c, s, b = oracle.quantize_uniform(x[i], lo[i], hi[i], 4, aux)
            assert np.array_equal(q.codes[i], c) and q.scales[i] == s and q.biases[i] == b
    for i in range(0, 300, 11):
        h = build_histogram(x[i], 50)
        want = oracle.build_histogram(x[i], 50)
        assert h.counts.tolist() == list(want[2]) and (h.lo, h.hi) == (want[0], want[1])
