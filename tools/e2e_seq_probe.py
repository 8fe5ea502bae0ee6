import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads
rows, DIM = 20_000_000, 64
dev = torch.device("cuda", 0)
x = workloads.mixed_table(rows, DIM, seed=1911, device=dev)
stride = eq.packed_row_stride(DIM, "fp16")
out = torch.empty(rows * stride, dtype=torch.uint8, device=dev)
st = torch.zeros(1, dtype=torch.int32, device=dev)
for _ in range(13):
    eq.quantize_pack_table4(x, "greedy", "fp16", 200, 0.16, out=out, status=st, check=False)
torch.cuda.synchronize()
xh = torch.empty((rows, DIM), dtype=torch.float32, pin_memory=True)
oh = torch.empty(rows * stride, dtype=torch.uint8, pin_memory=True)
xh.copy_(x)
table = eq.EmbeddingTable(xh.numpy())
mode = sys.argv[1] if len(sys.argv) > 1 else "keep"
if mode == "free":
    del x, out
    torch.cuda.empty_cache()
outh = oh.numpy()
for i in range(8):
    t0 = time.perf_counter(); eq.quantize_pack_table4(table, "greedy", "fp16", 200, 0.16, out=outh); t = time.perf_counter() - t0
    print(mode, i, round(t * 1e3, 1), flush=True)
