"""e2e host-pipeline timing for A/B runs (development probe): the public API on a pinned
20M x 64 table, 5 calls, min / median wall time.  Select the library with EQ4_LIB."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads
rows, d = 20_000_000, 64
x = workloads.mixed_table(rows, d, 1911)
xh = torch.empty((rows, d), dtype=torch.float32, pin_memory=True); xh.copy_(x)
del x; torch.cuda.empty_cache()
oh = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, pin_memory=True)
table = eq.EmbeddingTable(xh.numpy()); outh = oh.numpy()
eq.quantize_pack_table4(table, "greedy", "fp16", out=outh)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); eq.quantize_pack_table4(table, "greedy", "fp16", out=outh); ts.append(time.perf_counter() - t0)
ts = sorted(ts)
print(f"{os.environ.get('EQ4_LIB', 'tree')}: e2e min {ts[0]*1e3:.1f} ms  median {ts[2]*1e3:.1f} ms", flush=True)
