"""Break down the end-to-end (host buffers) path: raw pinned H2D / D2H bandwidth vs the
chunked eq4_quantize_pack_host pipeline at several chunk sizes (development probe)."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads, _lib

rows, d = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000, 64
x = workloads.mixed_table(rows, d, 1911)
xh = torch.empty((rows, d), dtype=torch.float32, pin_memory=True); xh.copy_(x)
stride = eq.packed_row_stride(d, "fp16")
oh = torch.empty(rows * stride, dtype=torch.uint8, pin_memory=True)
xd = torch.empty_like(x)
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter(); xd.copy_(xh, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter() - t0
print(f"H2D {xh.numel()*4/1e9:.2f} GB pinned: {t*1e3:.1f} ms = {xh.numel()*4/t/1e9:.1f} GB/s")
od = torch.empty(rows * stride, dtype=torch.uint8, device="cuda")
for _ in range(2):
    t0 = time.perf_counter(); oh.copy_(od, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter() - t0
print(f"D2H {od.numel()/1e9:.2f} GB pinned: {t*1e3:.1f} ms = {od.numel()/t/1e9:.1f} GB/s")
L = eq.load()
vp = ctypes.c_void_p
bad = np.full(1, -1, np.int64); blh = np.zeros(2)
for chunk_mb in (16, 64, 256):
    chunk_rows = (chunk_mb << 20) // (d * 4)
    for _ in range(2):
        t0 = time.perf_counter()
        rc = L.eq4_quantize_pack_host(vp(xh.data_ptr()), rows, d, d, 1, 200, 0.16, 1, vp(oh.data_ptr()),
                                      None, None, None, None, None, chunk_rows,
                                      bad.ctypes.data_as(vp), blh.ctypes.data_as(vp))
        t = time.perf_counter() - t0
    print(f"host pipeline chunk {chunk_mb} MiB: rc={rc} {t*1e3:.1f} ms = {rows/t/1e6:.1f} Mrows/s")
