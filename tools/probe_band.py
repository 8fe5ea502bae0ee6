"""A/B of the GREEDY near-boundary count zone (development probe): time + rare-path counters."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads, _lib

def timeit(fn, n=5, w=2):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n

for rows, d, dist in [(20_000_000, 64, "mixed"), (16_777_216, 16, "gauss"), (2_097_152, 128, "gauss")]:
    x = (workloads.mixed_table if dist == "mixed" else workloads.gaussian_table)(rows, d, 1)
    out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for sc in sys.argv[1:] or ["1", "0"]:
        os.environ["EQ4_DEV_KMISX_SCALE"] = sc
        f = lambda: eq.quantize_pack_table4(x, "greedy", "fp16", out=out, status=st, check=False)
        f(); torch.cuda.synchronize()
        _lib.diag_counters(reset=True)
        f(); torch.cuda.synchronize()
        dg = _lib.diag_counters(reset=True)
        ms = timeit(f)
        print(f"{rows}x{d} {dist} kmisx*{sc}: {ms:.3f} ms  {dg}", flush=True)
    del x, out
