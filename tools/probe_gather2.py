"""ncu target: torch.index_select gathers of 32 / 36 / 64-byte rows (1M random rows of 20M)."""
import torch
rows, nq = 20_000_000, 1 << 20
g = torch.Generator(device="cuda").manual_seed(1)
idx = torch.randint(0, rows, (nq,), device="cuda", generator=g)
for words in (8, 9, 16):
    t = torch.randint(0, 1 << 30, (rows, words), dtype=torch.int32, device="cuda")
    for _ in range(2):
        torch.index_select(t, 0, idx)
    torch.cuda.synchronize()
    del t
print("ok")
