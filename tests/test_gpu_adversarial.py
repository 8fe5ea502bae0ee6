"""GREEDY on adversarial rows (tests/adversarial.py, fixture tests/golden/adversarial.npz):
repeated values parked within eta of a code boundary of a candidate the walk visits, with
that iteration's two losses closer than the misrounds can move them.  The kernel must count
those elements (near_escalate) and re-decide in float64; bytes, ranges and iteration counts
bit-exact against the oracle."""

import numpy as np
import pytest
import torch

import oracle
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import _lib
from test_oracle_golden import _bits, _load

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [64, 16, 128])
def test_adversarial_rows_bit_exact(d):
    x = _load("adversarial.npz")[f"x_{d}"]
    for aux in ("fp16", "fp32"):
        _lib.diag_counters(reset=True)
        p, rr = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "greedy", aux, 200, 0.16,
                                        with_rows=True)
        diag = _lib.diag_counters(reset=True)
        want = oracle.quantize_pack_table(x, "greedy", 200, 0.16, aux)
        st = eq.packed_row_stride(d, aux)
        bad = np.nonzero((p.buffer.reshape(-1, st) != want.packed.reshape(-1, st)).any(1))[0]
        assert bad.size == 0, (aux, bad[:10], diag)
        assert np.array_equal(_bits(rr.xmin.cpu().numpy()), _bits(want.xmin))
        assert np.array_equal(_bits(rr.xmax.cpu().numpy()), _bits(want.xmax))
        assert np.array_equal(rr.info0.cpu().numpy(), want.info0)
        # the rows reach the counting path and some of them need the float64 decision
        assert diag["near_count_checks"] > 0 and diag["near_count_escalations"] > 0, diag


def test_adversarial_rows_masked_layout():
    """The same rows through the masked kernels (16-byte misaligned table view)."""
    x = _load("adversarial.npz")["x_64"][:3000]
    buf = torch.zeros(x.size + 1, dtype=torch.float32, device="cuda")
    buf[1:] = torch.from_numpy(x.reshape(-1)).cuda()
    xd = buf[1:].view(x.shape)
    p, rr = eq.quantize_pack_table4(xd, "greedy", "fp16", 200, 0.16, with_rows=True)
    want = oracle.quantize_pack_table(x, "greedy", 200, 0.16, "fp16")
    assert np.array_equal(p.buffer, want.packed)
    assert np.array_equal(rr.info0.cpu().numpy(), want.info0)
