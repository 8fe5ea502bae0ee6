"""Iterate the pooled-lookup golden cases of tests/golden/sls.npz (made by the reference)."""

import json
import os

import numpy as np

G = os.path.join(os.path.dirname(__file__), "golden")


def sls_cases():
    f = np.load(os.path.join(G, "sls.npz"))
    pb = po = pi = pl = 0
    for rows, d, aux16, batch, nidx in f["meta"]:
        rows, d, batch, nidx = int(rows), int(d), int(batch), int(nidx)
        aux = "fp16" if aux16 else "fp32"
        stride = (d + 1) // 2 + 2 * (2 if aux16 else 4)
        packed = f["packed"][pb:pb + rows * stride]
        out = f["out"][po:po + batch * d].reshape(batch, d)
        idx = f["indices"][pi:pi + nidx]
        ln = f["lengths"][pl:pl + batch]
        pb += rows * stride; po += batch * d; pi += nidx; pl += batch
        yield packed, rows, d, aux, idx, ln, out


def sls_errors():
    return json.loads(str(np.load(os.path.join(G, "sls.npz"))["errors"]))
