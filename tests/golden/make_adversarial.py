"""Generate tests/golden/adversarial.npz: adversarial GREEDY rows (tests/adversarial.py).

    python tests/golden/make_adversarial.py [rows_d64] [procs]

Inputs only -- the expected outputs are the oracle's on the same rows at test time (the
oracle is pinned to the reference by tests/test_oracle_golden.py).  Deterministic: each
chunk of rows has its own seed.
"""

from __future__ import annotations

import os
import sys
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

from adversarial import adversarial_table  # noqa: E402

CHUNK = 250


def _chunk(args):
    d, seed = args
    return adversarial_table(CHUNK, d, seed)


def make(rows_by_d, procs):
    out = {}
    with Pool(procs) as pool:
        for d, rows in rows_by_d.items():
            jobs = [(d, 1911 * 1000 + d * 100 + c) for c in range(rows // CHUNK)]
            out[f"x_{d}"] = np.concatenate(pool.map(_chunk, jobs))
            print(f"d={d}: {out[f'x_{d}'].shape[0]} rows", flush=True)
    return out


if __name__ == "__main__":
    n64 = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
    procs = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
    out = make({64: n64, 16: 2000, 128: 2000}, procs)
    np.savez_compressed(os.path.join(HERE, "adversarial.npz"), **out)
