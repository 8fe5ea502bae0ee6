"""GREEDY rare-path counters (deferred rows, exact re-decisions, near-boundary counts) with and
without the exact pass:  python tools/greedy_deferrals.py rows:d:dist ..."""
import os, sys; sys.path.insert(0, '.')
import torch, paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads, _lib
for c in sys.argv[1:]:
    rows, d, dist = c.split(":"); rows, d = int(rows), int(d)
    x = (workloads.mixed_table if dist == "mixed" else workloads.gaussian_table)(rows, d, 7)
    out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    for skip in (True, False):
        if skip: os.environ["EQ4_DEV_SKIP_EXACT"] = "1"
        else: os.environ.pop("EQ4_DEV_SKIP_EXACT", None)
        _lib.diag_counters(reset=True)
        eq.quantize_pack_table4(x, "greedy", "fp16", 200, 0.16, out=out, check=False)
        torch.cuda.synchronize()
        print(c, "skip" if skip else "full", _lib.diag_counters(reset=True), flush=True)
