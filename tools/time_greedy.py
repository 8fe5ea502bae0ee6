"""GREEDY device time of the two-pass path and of the screening kernel alone (EQ4_DEV_SKIP_EXACT),
for A/B of library variants (EQ4_LIB=variants/libeq4_NAME.so):  python tools/time_greedy.py rows:d:dist ..."""
import os, sys; sys.path.insert(0, '.')
import torch, paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads
def timeit(fn, n=5, w=2):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
lib = os.path.basename(os.environ.get("EQ4_LIB", "in-tree"))
for c in sys.argv[1:]:
    rows, d, dist = c.split(":"); rows, d = int(rows), int(d)
    x = (workloads.mixed_table if dist == "mixed" else workloads.gaussian_table)(rows, d, 1)
    out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    f = lambda: eq.quantize_pack_table4(x, "greedy", "fp16", 200, 0.16, out=out, status=st, check=False)
    os.environ.pop("EQ4_DEV_SKIP_EXACT", None)
    full = timeit(f)
    os.environ["EQ4_DEV_SKIP_EXACT"] = "1"
    fast = timeit(f)
    os.environ.pop("EQ4_DEV_SKIP_EXACT", None)
    print(f"{lib} {c}: two-pass {full:.3f} ms, screen only {fast:.3f} ms", flush=True)
    del x, out
