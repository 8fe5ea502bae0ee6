"""Time the streamed EMBT -> EMBQ pipeline (quantize_file) at north-star size (development probe)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
d = 64
base = sys.argv[2] if len(sys.argv) > 2 else "/dev/shm"
src, dst = os.path.join(base, "t.embt"), os.path.join(base, "t.embq")
x = workloads.mixed_table(rows, d, 1911)
t0 = time.perf_counter()
eq.write_embt(src, x.cpu().numpy())
print(f"write_embt {rows}x{d}: {time.perf_counter()-t0:.2f} s", flush=True)
del x
torch.cuda.empty_cache()
for chunk in (0, 1 << 20, 1 << 22):
    for _ in range(2):
        t0 = time.perf_counter()
        eq.quantize_file(src, dst, "greedy", "fp16", chunk_rows=chunk)
        t = time.perf_counter() - t0
    print(f"quantize_file greedy fp16 chunk_rows={chunk}: {t*1e3:.1f} ms  {rows/t/1e6:.1f} Mrows/s  "
          f"{(os.path.getsize(src))/t/1e9:.1f} GB/s in", flush=True)
os.remove(src); os.remove(dst)
