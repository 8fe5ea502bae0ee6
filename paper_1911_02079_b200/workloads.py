"""Seeded synthetic tables on the GPU (BASELINE.json configs).

The paper's trained Criteo tables are not available; these
generators stand in with the shapes and value distributions BASELINE.json
names.  All draws come from a seeded ``torch.Generator(device="cuda")``.
"""

from __future__ import annotations

import math

import torch


def gaussian_table(rows: int, dim: int, seed: int, device="cuda") -> torch.Tensor:
    """Configs 2, 4, 5a: i.i.d. N(0, 1) float32."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn(rows, dim, generator=g, device=device, dtype=torch.float32)


def mixed_table(rows: int, dim: int, seed: int, device="cuda", chunk: int = 1 << 20) -> torch.Tensor:
    """Configs 3 and 5b ("mimicking trained embeddings"), per row:
    s ~ LogNormal(mu=-2, sigma=1); offset ~ N(0, (0.1 s)^2);
    family = row % 3 -> N(0, s^2) | U[-sqrt(3) s, sqrt(3) s] | s * t_3
    (t_3 = Z / sqrt(chi2_3 / 3), chi2_3 = sum of three squared normals)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty(rows, dim, device=device, dtype=torch.float32)
    for r0 in range(0, rows, chunk):
        n = min(chunk, rows - r0)
        s = torch.exp(torch.randn(n, 1, generator=g, device=device) - 2.0)
        off = torch.randn(n, 1, generator=g, device=device) * 0.1 * s
        fam = (torch.arange(r0, r0 + n, device=device) % 3).unsqueeze(1)
        z = torch.randn(n, dim, generator=g, device=device)
        u = (torch.rand(n, dim, generator=g, device=device) * 2.0 - 1.0) * math.sqrt(3.0)
        chi = (torch.randn(n, dim, 3, generator=g, device=device) ** 2).sum(-1)
        t3 = torch.randn(n, dim, generator=g, device=device) / torch.sqrt(chi / 3.0)
        x = torch.where(fam == 0, z, torch.where(fam == 1, u, t3))
        out[r0:r0 + n] = x * s + off
    return out
