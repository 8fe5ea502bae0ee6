"""KMEANS rows and HIST-APPRX device time (A/B of library variants via EQ4_LIB)."""
import os, sys; sys.path.insert(0, '.')
import torch, paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads
from paper_1911_02079_b200.codebook import kmeans_rows, kmeans_row_stride
def timeit(fn, n=5, w=2):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
lib = os.path.basename(os.environ.get("EQ4_LIB", "in-tree"))
for rows, d in ((262144, 128), (1048576, 64)):
    x = workloads.gaussian_table(rows, d, 7)
    kout = torch.empty(rows * kmeans_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    kit = torch.empty(rows, dtype=torch.int32, device="cuda")
    ms_k = timeit(lambda: kmeans_rows(x, "fp16", out=kout, iters=kit, check=False))
    out = torch.empty(16384 * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    ms_h = timeit(lambda: eq.quantize_pack_table4(x[:16384], "hist-apprx", "fp16", 200, out=out, check=False))
    print(f"{lib} kmeans {rows}x{d}: {ms_k:.3f} ms   hist-apprx 16384x{d}: {ms_h:.3f} ms", flush=True)
