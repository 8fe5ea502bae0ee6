"""Quick device-side timing of the fused kernels (development probe, not the bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads

def timeit(fn, n=5, w=2):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n

cases = sys.argv[1:] or ["greedy:20000000:64:mixed", "asym:4194304:64:gauss", "greedy:4194304:128:mixed"]
for c in cases:
    m, rows, d, dist = c.split(":"); rows, d = int(rows), int(d)
    x = (workloads.mixed_table if dist == "mixed" else workloads.gaussian_table)(rows, d, 1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    rr = eq.RowResults(None, None, torch.empty(rows, dtype=torch.int32, device="cuda"), None, None)
    f = lambda: eq.quantize_pack_table4(x, m, "fp16", out=out, status=st, check=False, rows_out=rr)
    ms = timeit(f)
    it = rr.info0.double()
    evals = torch.where(it >= 0, 1 + 2 * it, torch.zeros_like(it)).sum().item()
    flop = 13.0 * d * evals
    byt = rows * (4 * d + (d + 1) // 2 + 4)
    print(f"{c}: {ms:.3f} ms  {rows/ms/1e6:.3f} Grows/s  {byt/ms/1e6:.1f} GB/s  {flop/ms/1e9:.2f} TFLOP/s(alg) status={st.item()}", flush=True)
