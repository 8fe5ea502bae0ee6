"""INTEGRATION.md's reference-side binding, executed: the `embquant/_eq4.py` block is
extracted from the document, installed into a scratch `embquant` package (its `packed` and
`clipping` imports bound to this repo's PackedTable4 / WorkCounters, which mirror the
reference's), pointed at the built libeq4.so, and called like the reference would call it.
The packed bytes must equal the oracle's."""

import importlib
import os
import re
import sys

import numpy as np
import pytest

import oracle
import paper_1911_02079_b200 as eq
from oracle import rng

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _binding_source() -> str:
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    head = doc.index("`embquant/_eq4.py`")
    m = re.search(r"```python\n(.*?)```", doc[head:], re.S)
    assert m, "INTEGRATION.md lost its _eq4.py block"
    return m.group(1)


@pytest.fixture(scope="module")
def binding(tmp_path_factory):
    pkg = tmp_path_factory.mktemp("refpkg") / "embquant"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "packed.py").write_text("from paper_1911_02079_b200.api import PackedTable4\n")
    (pkg / "clipping.py").write_text("from paper_1911_02079_b200.api import WorkCounters\n")
    src = _binding_source().replace('ctypes.CDLL("libeq4.so")', f'ctypes.CDLL({eq.LIB_PATH!r})')
    (pkg / "_eq4.py").write_text(src)
    sys.path.insert(0, str(pkg.parent))
    try:
        for name in [n for n in sys.modules if n == "embquant" or n.startswith("embquant.")]:
            del sys.modules[name]
        yield importlib.import_module("embquant._eq4")
    finally:
        sys.path.remove(str(pkg.parent))
        for name in [n for n in sys.modules if n == "embquant" or n.startswith("embquant.")]:
            del sys.modules[name]


@pytest.mark.parametrize("method,b", [("greedy", 200), ("asym", 200), ("hist-brute", 64), ("gss", 200),
                                      ("aciq", 200), ("sym", 200)])
def test_integration_binding_matches_oracle(binding, method, b):
    x = rng.mixed_table(3000 if method != "hist-brute" else 400, 48, 17)
    t = eq.EmbeddingTable(x)
    for aux in ("fp16", "fp32"):
        c = eq.WorkCounters()
        p = binding.quantize_pack(t, method, aux, b, 0.16, c)
        want = oracle.quantize_pack_table(x, method, b, 0.16, aux)
        assert np.array_equal(np.asarray(p.buffer), want.packed), (method, aux)
        if method == "greedy":
            assert c.loss_evals == int(np.sum(np.where(want.info0 < 0, 0, 1 + 2 * want.info0.astype(np.int64))))


def test_integration_binding_raises_reference_error(binding):
    """A GREEDY walk whose candidates cross (b=200, r=1.0): the reference's ClipRange
    ValueError text (golden edge case 'b200_r1.0')."""
    import json

    f = np.load(os.path.join(ROOT, "tests", "golden", "edge.npz"))
    meta = json.loads(str(f["meta"]))
    k = next(i for i, m in enumerate(meta) if m["name"] == "b200_r1.0")
    with pytest.raises(ValueError, match=re.escape(meta[k]["greedy_error"])):
        binding.quantize_pack(eq.EmbeddingTable(f[f"x_{k}"]), "greedy", "fp16", 200, 1.0, None)
