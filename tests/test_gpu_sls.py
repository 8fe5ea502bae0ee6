"""GPU parity of the pooled lookup over packed rows (sparse_lengths_sum_4bit, packed.py:167-177)
against fixtures from the reference and the C oracle (packed.py:202-221 restated): bit-exact."""

import numpy as np
import pytest
import torch

import oracle
import paper_1911_02079_b200 as eq
from sls_cases import sls_cases, sls_errors

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_sls_golden_cases_bit_exact():
    n = 0
    for packed, rows, d, aux, idx, ln, want in sls_cases():
        p = eq.PackedTable4(rows, d, aux, buffer=packed)
        got = eq.sparse_lengths_sum_4bit(p, eq.PooledQuery(idx, ln))
        assert got.shape == want.shape
        assert np.array_equal(_bits(got), _bits(want)), (n, rows, d, aux)
        n += 1
    assert n == 400


def test_sls_error_texts_match_reference():
    errs = sls_errors()
    p = eq.pack_table4(eq.UniformQuantTable(np.zeros((4, 6), np.uint8), np.ones(4), np.zeros(4), 4,
                                            "fp16"))
    with pytest.raises(IndexError) as e:
        eq.sparse_lengths_sum_4bit(p, eq.PooledQuery([0, 1, 9], [3]))
    assert f"IndexError: {e.value}" == errs["oob"]
    with pytest.raises(ValueError) as e:
        eq.PooledQuery([0, 1], [-1, 2])
    assert f"ValueError: {e.value}" == errs["neg"]
    with pytest.raises(ValueError) as e:
        eq.PooledQuery([1, 2], [1])
    assert f"ValueError: {e.value}" == errs["sum"]
    # device queries are validated by the kernel with the same texts
    dev = torch.device("cuda")
    with pytest.raises(IndexError, match="query index 9 at position 2 out of range for 4 rows"):
        eq.sparse_lengths_sum_4bit(p, eq.PooledQuery(torch.tensor([0, 1, 9], device=dev),
                                                     torch.tensor([3], device=dev)))
    with pytest.raises(ValueError, match="lengths must be non-negative"):
        eq.sparse_lengths_sum_4bit(p, eq.PooledQuery(torch.tensor([0, 1], device=dev),
                                                     torch.tensor([-1, 2], device=dev)))
    with pytest.raises(ValueError, match="lengths sum to 1 but there are 2 indices"):
        eq.sparse_lengths_sum_4bit(p, eq.PooledQuery(torch.tensor([1, 2], device=dev),
                                                     torch.tensor([1], device=dev)))


def test_sls_first_bad_position_among_many():
    p = eq.pack_table4(eq.UniformQuantTable(np.zeros((10, 64), np.uint8), np.ones(10), np.zeros(10),
                                            4, "fp32"))
    rng = np.random.default_rng(3)
    idx = rng.integers(0, 10, size=5000)
    idx[[1234, 2000, 4999]] = [-1, 10, 99]
    ln = np.full(50, 100)
    with pytest.raises(IndexError, match="query index -1 at position 1234 out of range"):
        eq.sparse_lengths_sum_4bit(p, eq.PooledQuery(idx, ln))


@pytest.mark.parametrize("d", [1, 7, 8, 16, 24, 32, 33, 40, 64, 96, 128, 200, 256, 512, 1000, 1024,
                               2048])
@pytest.mark.parametrize("aux", ["fp16", "fp32"])
def test_sls_random_vs_oracle(d, aux):
    rng = np.random.default_rng(d * 7 + (aux == "fp16"))
    rows = 3000
    x = (rng.standard_normal((rows, d)) * rng.uniform(0.01, 5, size=(rows, 1))).astype(np.float32)
    p, _ = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "asym", aux)
    batch = 700
    ln = rng.integers(0, 40, size=batch)
    ln[::37] = 0
    idx = rng.integers(0, rows, size=int(ln.sum()))
    got = eq.sparse_lengths_sum_4bit(p, eq.PooledQuery(idx, ln))
    want, rc, _ = oracle.sparse_lengths_sum4(p.buffer, rows, d, aux, idx, ln)
    assert rc == 0
    assert np.array_equal(_bits(got), _bits(want))


def test_sls_device_query_and_out():
    rng = np.random.default_rng(5)
    x = torch.randn(10000, 64, device="cuda")
    p, _ = eq.quantize_pack_table4(x, "greedy", "fp16")
    ln = torch.randint(0, 64, (1024,), device="cuda")
    idx = torch.randint(0, 10000, (int(ln.sum()),), device="cuda")
    out = torch.empty(1024, 64, device="cuda")
    got = eq.sparse_lengths_sum_4bit(p, eq.PooledQuery(idx, ln), out=out)
    assert got.data_ptr() == out.data_ptr()
    want, rc, _ = oracle.sparse_lengths_sum4(p.buffer, 10000, 64, "fp16", idx.cpu().numpy(),
                                             ln.cpu().numpy())
    assert rc == 0 and np.array_equal(_bits(got.cpu().numpy()), _bits(want))
    # empty batch and all-empty segments
    assert eq.sparse_lengths_sum_4bit(p, eq.PooledQuery([], [])).shape == (0, 64)
    z = eq.sparse_lengths_sum_4bit(p, eq.PooledQuery([], [0, 0, 0]))
    assert z.shape == (3, 64) and not z.any()
