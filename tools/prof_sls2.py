"""Pooled lookup with long segments (batch 1024 x pool 1024) as an ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
rows = 20_000_000
x = torch.randn(rows, 64, device="cuda")
p, _ = eq.quantize_pack_table4(x, "asym", "fp16")
del x
g = torch.Generator(device="cuda").manual_seed(1)
batch, pool = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, int(sys.argv[2]) if len(sys.argv) > 2 else 1024
idx = torch.randint(0, rows, (batch * pool,), device="cuda", generator=g)
ln = torch.full((batch,), pool, dtype=torch.int64, device="cuda")
q = eq.PooledQuery(idx, ln)
for _ in range(2):
    eq.sparse_lengths_sum_4bit(p, q, check=False)
torch.cuda.synchronize()
print("ok")
