"""Device timing of row-wise KMEANS (development probe): rows:d cases, N(0,1) rows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_02079_b200.codebook import kmeans_rows, kmeans_row_stride
for c in sys.argv[1:] or ["1048576:64"]:
    rows, d = map(int, c.split(":"))
    x = torch.randn(rows, d, device="cuda")
    out = torch.empty(rows * kmeans_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    it = torch.empty(rows, dtype=torch.int32, device="cuda")
    kmeans_rows(x, "fp16", out=out, iters=it)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); kmeans_rows(x, "fp16", out=out, iters=it, check=False); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"kmeans {rows}x{d}: {ms:.2f} ms  {rows/ms/1e3:.2f} M rows/s  mean Lloyd rounds "
          f"{it.clamp(min=0).float().mean().item():.1f}", flush=True)
