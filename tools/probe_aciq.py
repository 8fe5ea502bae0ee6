"""ACIQ: cooperative k_aciq8 vs the lane-per-row k_rowrange (EQ4_DEV_ACIQ_LANE): device time and
identical bytes / ranges (development probe).  python tools/probe_aciq.py [rows:d ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads


def timeit(fn, n=20, w=3):
    for _ in range(w): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n


for c in sys.argv[1:] or ["4194304:64", "4194304:32", "2097152:128", "8388608:16", "4194304:8"]:
    rows, d = map(int, c.split(":"))
    x = workloads.gaussian_table(rows, d, 7)
    res = {}
    for mode in ("lane", "coop"):
        if mode == "lane": os.environ["EQ4_DEV_ACIQ_LANE"] = "1"
        else: os.environ.pop("EQ4_DEV_ACIQ_LANE", None)
        out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
        rr = eq.RowResults(torch.empty(rows, dtype=torch.float64, device="cuda"),
                           torch.empty(rows, dtype=torch.float64, device="cuda"), None, None, None)
        eq.quantize_pack_table4(x, "aciq", "fp16", out=out, rows_out=rr)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        ms = timeit(lambda: eq.quantize_pack_table4(x, "aciq", "fp16", out=out, status=st, check=False))
        res[mode] = (ms, out, rr)
    os.environ.pop("EQ4_DEV_ACIQ_LANE", None)
    same = (torch.equal(res["lane"][1], res["coop"][1]) and torch.equal(res["lane"][2].xmin, res["coop"][2].xmin)
            and torch.equal(res["lane"][2].xmax, res["coop"][2].xmax))
    byt = rows * (4 * d + d // 2 + 4)
    print(f"aciq {c}: lane {res['lane'][0]:.4f} ms  coop {res['coop'][0]:.4f} ms  "
          f"({byt / res['coop'][0] / 1e6:.0f} GB/s)  identical={same}", flush=True)
