"""A/B of the GREEDY screens on wide rows: the table walk (k_greedy_table) against the per-element
screen (k_greedy_fast), 1 GiB N(0,1) tables, with deferral counts and a byte comparison of the two.
    python tools/probe_table_walk.py [d ...]"""
import os, sys; sys.path.insert(0, '.')
import torch, paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads, _lib
def timeit(fn, n=5, w=2):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
ds = [int(a) for a in sys.argv[1:]] or [512, 1024, 2048, 4096, 8192, 16384]
for d in ds:
    rows = (1 << 28) // d
    x = workloads.gaussian_table(rows, d, 1)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = {}
    for name, min_d in (("table", 16), ("elem", 1 << 20)):
        os.environ["EQ4_DEV_TABLE_MIN_D"] = str(min_d)
        out = torch.zeros(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
        f = lambda: eq.quantize_pack_table4(x, "greedy", "fp16", 200, 0.16, out=out, status=st, check=False)
        _lib.diag_counters(reset=True)
        f(); torch.cuda.synchronize()
        dg = _lib.diag_counters(reset=True)
        full = timeit(f)
        os.environ["EQ4_DEV_SKIP_EXACT"] = "1"
        fast = timeit(f)
        os.environ.pop("EQ4_DEV_SKIP_EXACT", None)
        f(); torch.cuda.synchronize()
        res[name] = (full, fast, dg["deferred_rows"], out)
    same = torch.equal(res["table"][3], res["elem"][3])
    print(f"d={d} rows={rows}: table {res['table'][0]:.3f} ms (screen {res['table'][1]:.3f}, deferred {res['table'][2]})"
          f" | elem {res['elem'][0]:.3f} ms (screen {res['elem'][1]:.3f}, deferred {res['elem'][2]}) | same bytes {same}", flush=True)
    del x
os.environ.pop("EQ4_DEV_TABLE_MIN_D", None)
