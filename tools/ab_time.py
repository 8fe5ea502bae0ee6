"""A/B device time of GREEDY launches between libeq4.so builds (development probe).
    EQ4_LIB=path python tools/ab_time.py rows:d:dist ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
import paper_1911_02079_b200.api
from paper_1911_02079_b200 import workloads

def timeit(fn, n=5, w=2):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n

lib = os.environ.get("EQ4_LIB", "in-tree")
for c in sys.argv[1:] or ["20000000:64:mixed", "16777216:16:gauss", "2097152:128:gauss"]:
    rows, d, dist = c.split(":"); rows, d = int(rows), int(d)
    x = (workloads.mixed_table if dist == "mixed" else workloads.gaussian_table)(rows, d, 1)
    out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    import ctypes
    L = ctypes.CDLL(os.environ.get("EQ4_LIB") or eq.LIB_PATH)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.eq4_quantize_pack.argtypes = [vp, i64, i64, i64, i32, i32, dbl, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    f = lambda: L.eq4_quantize_pack(eq.api._vp(x), rows, d, d, 1, 200, 0.16, 1, eq.api._vp(out), None, None,
                                    None, None, None, eq.api._vp(st), eq.api._stream_handle())
    print(f"{os.path.basename(lib)} {c}: {timeit(f):.3f} ms", flush=True)
    del x, out
