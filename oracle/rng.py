"""Seeded table generator restated from the reference's rng.py -- TEST INFRASTRUCTURE.

The reference draws synthetic tables from a counter-based splitmix64 stream
(rng.py:20-52): output i mixes ``seed + (i+1)*golden`` through the public
splitmix64 finaliser; uniforms in (0,1) take the top 53 bits plus a half ulp;
gaussians use Box-Muller on consecutive uniform pairs (rng.py:79-87) and
laplacians the inverse CDF (rng.py:90-92); the float64 stream is cast to
float32 (rng.py:95-104).  This port lets tests rebuild config-1 inputs
(``sample_table(gaussian(0,1), 10000, 64)``) without the reference; it is
pinned by the sha256 digests stored in tests/golden/config1.npz.
"""

from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX_A = np.uint64(0xBF58476D1CE4E5B9)
MIX_B = np.uint64(0x94D049BB133111EB)


def _finalise(z: np.ndarray) -> np.ndarray:
    """splitmix64 output function (xor-shift-multiply x2, xor-shift)."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * MIX_A
        z = (z ^ (z >> np.uint64(27))) * MIX_B
        return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, n: int) -> np.ndarray:
    """Outputs 1..n of the counter-based stream (rng.py:33-37)."""
    ctr = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _finalise(np.uint64(seed & _M64) + ctr * GOLDEN)


def uniform_open01(seed: int, n: int) -> np.ndarray:
    """n doubles strictly inside (0,1) from the top 53 bits (rng.py:40-43)."""
    top = (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64)
    return (top + 0.5) * (2.0 ** -53)


def derive_seed(seed: int, *salts: int) -> int:
    """Salt folding used by the reference sweeps and acceptance corpora (rng.py:46-52)."""
    s = np.uint64(seed & _M64)
    with np.errstate(over="ignore"):
        for salt in salts:
            s = _finalise(s + GOLDEN + np.uint64(salt & _M64) * MIX_A)
    return int(s)


def _gaussian(seed: int, n: int, loc: float, scale: float) -> np.ndarray:
    m = (n + 1) // 2
    u = uniform_open01(seed, 2 * m)
    rad = np.sqrt(-2.0 * np.log(u[0::2]))
    ang = 2.0 * np.pi * u[1::2]
    z = np.empty(2 * m)
    z[0::2] = rad * np.cos(ang)
    z[1::2] = rad * np.sin(ang)
    return loc + scale * z[:n]


def _laplacian(seed: int, n: int, loc: float, scale: float) -> np.ndarray:
    v = uniform_open01(seed, n) - 0.5
    return loc - scale * np.sign(v) * np.log1p(-2.0 * np.abs(v))


def sample_table(distribution: str, loc: float, scale: float, seed: int, rows: int,
                 dim: int) -> np.ndarray:
    """(rows, dim) float32 table, equal to the reference's sample_table(...).values."""
    if distribution not in ("gaussian", "laplacian"):
        raise ValueError(f"unknown distribution {distribution!r}")
    if rows < 1 or dim < 1:
        raise ValueError(f"rows and dim must be >= 1, got {rows}x{dim}")
    gen = _gaussian if distribution == "gaussian" else _laplacian
    return gen(seed, rows * dim, loc, scale).astype(np.float32).reshape(rows, dim)


def gaussian_row(seed: int, d: int, mean: float = 0.0, std: float = 1.0) -> np.ndarray:
    """The reference tests' ``oracles.gaussian_row`` (pkg/tests/oracles.py:18-19)."""
    return sample_table("gaussian", mean, std, seed, 1, d)[0]


def laplacian_row(seed: int, d: int, loc: float = 0.0, scale: float = 1.0) -> np.ndarray:
    return sample_table("laplacian", loc, scale, seed, 1, d)[0]


def mixed_table(rows: int, dim: int, seed: int) -> np.ndarray:
    """Config-3 style 'trained embedding' rows on the CPU (numpy Generator).

    Per row: s ~ LogNormal(-2, 1); offset ~ N(0, (0.1 s)^2); family = row % 3 ->
    N(0, s^2), U[-sqrt(3) s, sqrt(3) s], s * t_3.  The GPU bench uses the same
    recipe with torch's CUDA generator (paper_1911_02079_b200.workloads).
    """
    g = np.random.default_rng(seed)
    s = np.exp(g.normal(-2.0, 1.0, size=(rows, 1)))
    off = g.normal(0.0, 1.0, size=(rows, 1)) * 0.1 * s
    fam = (np.arange(rows) % 3)[:, None]
    z = g.normal(size=(rows, dim))
    u = g.uniform(-1.0, 1.0, size=(rows, dim)) * np.sqrt(3.0)
    chi = (g.normal(size=(rows, dim, 3)) ** 2).sum(-1)
    t3 = g.normal(size=(rows, dim)) / np.sqrt(chi / 3.0)
    x = np.where(fam == 0, z, np.where(fam == 1, u, t3)) * s + off
    return x.astype(np.float32)
