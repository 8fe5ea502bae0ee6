"""GREEDY two-pass (screen + deferred exact) vs one-pass k_greedy: device time, identical
bytes/ranges/iterations, deferred-row count (development probe).
    python tools/probe_two_pass.py [rows:d:dist ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads, _lib


def timeit(fn, n=5, w=2):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n


def run(x, one_pass):
    if one_pass:
        os.environ["EQ4_DEV_ONE_PASS"] = "1"
    else:
        os.environ.pop("EQ4_DEV_ONE_PASS", None)
    rows, d = x.shape
    out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rr = eq.RowResults(torch.empty(rows, dtype=torch.float64, device="cuda"),
                       torch.empty(rows, dtype=torch.float64, device="cuda"),
                       torch.empty(rows, dtype=torch.int32, device="cuda"),
                       torch.empty(rows, dtype=torch.int32, device="cuda"), None)
    _lib.diag_counters(reset=True)
    eq.quantize_pack_table4(x, "greedy", "fp16", 200, 0.16, out=out, rows_out=rr, status=st, check=False)
    torch.cuda.synchronize()
    diag = _lib.diag_counters(reset=True)
    f = lambda: eq.quantize_pack_table4(x, "greedy", "fp16", 200, 0.16, out=out, status=st, check=False)
    ms = timeit(f)
    return ms, out, rr, diag, int(st.item())


for c in sys.argv[1:] or ["20000000:64:mixed", "4194304:128:mixed", "16777216:16:gauss",
                          "8388608:32:gauss", "4194304:64:gauss", "2097152:128:gauss", "262144:1024:gauss",
                          "65536:4096:gauss"]:
    rows, d, dist = c.split(":"); rows, d = int(rows), int(d)
    x = (workloads.mixed_table if dist == "mixed" else workloads.gaussian_table)(rows, d, 1)
    m1, o1, r1, d1, s1 = run(x, True)
    m2, o2, r2, d2, s2 = run(x, False)
    same = (torch.equal(o1, o2) and torch.equal(r1.xmin, r2.xmin) and torch.equal(r1.xmax, r2.xmax)
            and torch.equal(r1.info0, r2.info0) and torch.equal(r1.info1, r2.info1) and s1 == s2)
    print(f"{c}: one-pass {m1:.3f} ms  two-pass {m2:.3f} ms  ({m1 / m2:.3f}x)  identical={same}  "
          f"deferred={d2['deferred_rows']} ({100 * d2['deferred_rows'] / rows:.2f}%)  "
          f"redecisions one/two={d1['exact_redecisions']}/{d2['exact_redecisions']}", flush=True)
    del x, o1, o2, r1, r2
    torch.cuda.empty_cache()
