"""GPU parity of row-wise KMEANS codebooks (codebook.py:35-172) against reference-made fixtures
(tests/golden/kmeans.npz: codebooks, indices and EMBQ kmeans_row files) and the C oracle."""

import numpy as np
import pytest
import torch

import oracle
import paper_1911_02079_b200 as eq
from oracle import rng
from test_oracle_golden import KMEANS_TABLES, _load

pytestmark = pytest.mark.gpu


def test_kmeans_golden_codebooks_indices_and_files(tmp_path):
    f = _load("kmeans.npz")
    for tname in KMEANS_TABLES:
        x = f[f"x_{tname}"]
        for aux in ("fp16", "fp32"):
            q = eq.quantize_table(x, "kmeans", 4, aux)
            assert isinstance(q, eq.CodebookQuantTable)
            assert np.array_equal(q.codebooks.view(np.uint8), f[f"books_{tname}_{aux}"].view(np.uint8)), (tname, aux)
            assert np.array_equal(q.indices, f[f"idx_{tname}_{aux}"]), (tname, aux)
            path = tmp_path / f"{tname}_{aux}.embq"
            eq.write_embq(path, q)
            assert path.read_bytes() == f[f"embq_{tname}_{aux}"].tobytes(), (tname, aux)
            back = eq.read_embq(path)
            assert np.array_equal(back.indices, q.indices)
            assert np.array_equal(back.dequantize(), q.dequantize())


@pytest.mark.parametrize("rows,d,gen", [(5000, 64, "gauss"), (3000, 17, "mixed"), (800, 128, "mixed"),
                                        (300, 256, "gauss"), (2000, 8, "lap"), (500, 3, "gauss")])
@pytest.mark.parametrize("aux", ["fp16", "fp32"])
def test_kmeans_random_vs_oracle(rows, d, gen, aux):
    if gen == "mixed":
        x = rng.mixed_table(rows, d, d + 1)
    else:
        x = rng.sample_table("laplacian" if gen == "lap" else "gaussian", 0.0, 1.0, d + 2, rows, d)
    x[::97] = np.round(x[::97] * 2) / 2          # rows with few distinct values (shortcut path)
    it = torch.empty(rows, dtype=torch.int32, device="cuda")
    from paper_1911_02079_b200.codebook import CodebookQuantTable, kmeans_rows

    payload = kmeans_rows(torch.from_numpy(x).cuda(), aux, iters=it).cpu().numpy()
    q = CodebookQuantTable.from_payload(payload, rows, d, aux)
    books, idx, its = oracle.kmeans_table(x, aux)
    assert np.array_equal(q.codebooks.view(np.uint8), books.view(np.uint8))
    assert np.array_equal(q.indices, idx)
    assert np.array_equal(it.cpu().numpy(), its)


def test_kmeans_nonfinite():
    from paper_1911_02079_b200.codebook import kmeans_rows

    x = torch.randn(64, 32, device="cuda")
    x[5, 3] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        kmeans_rows(x, "fp16")


@pytest.mark.parametrize("d,rows", [(249, 64), (250, 64), (255, 40), (257, 40), (300, 40), (640, 16), (1000, 8)])
def test_kmeans_pairwise_leaves_and_wide_rows(d, rows):
    """Rows whose SSE / cluster-mean sums split into more than two numpy leaves (d or a
    cluster of 249..255 elements: the right half of 129..135 splits again) and rows wider
    than 256: codebooks, indices and Lloyd rounds bit-exact against the oracle."""
    from paper_1911_02079_b200.codebook import kmeans_rows

    x = rng.mixed_table(rows, d, d)
    x[0, : d - 3] = x[0, 0]            # one cluster holding all but 3 elements
    x[1, : d // 2] = 1.0 + np.arange(d // 2, dtype=np.float32) * 1e-6
    for aux in ("fp16", "fp32"):
        it = torch.empty(rows, dtype=torch.int32, device="cuda")
        payload = kmeans_rows(torch.from_numpy(x).cuda(), aux, iters=it).cpu().numpy()
        from paper_1911_02079_b200.codebook import CodebookQuantTable

        q = CodebookQuantTable.from_payload(payload, rows, d, aux)
        books, idx, its = oracle.kmeans_table(x, aux)
        assert np.array_equal(q.codebooks.view(np.uint8), books.view(np.uint8)), (d, aux)
        assert np.array_equal(q.indices, idx), (d, aux)
        assert np.array_equal(it.cpu().numpy(), its), (d, aux)
