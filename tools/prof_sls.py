"""One pooled lookup (20M x 64 fp16, batch 16384 x pool 64) + one torch index_select of 36-byte rows,
as ncu targets."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
rows = 20_000_000
x = torch.randn(rows, 64, device="cuda")
p, _ = eq.quantize_pack_table4(x, "asym", "fp16")
del x
g = torch.Generator(device="cuda").manual_seed(1)
idx = torch.randint(0, rows, (16384 * 64,), device="cuda", generator=g)
ln = torch.full((16384,), 64, dtype=torch.int64, device="cuda")
q = eq.PooledQuery(idx, ln)
for _ in range(2):
    eq.sparse_lengths_sum_4bit(p, q, check=False)
t = p.device_buffer.view(torch.int32).view(rows, 9)
for _ in range(2):
    torch.index_select(t, 0, idx)
torch.cuda.synchronize()
print("ok")
