"""Launch each hot kernel a few times (target for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads
which = sys.argv[1:] or ["asym", "greedy"]
for w in which:
    if w == "asym":
        x = workloads.gaussian_table(4_194_304, 64, 7)
        m = "asym"
    else:
        x = workloads.mixed_table(2_000_000, 64, 7)
        m = "greedy"
    out = torch.empty(x.shape[0] * 36, dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        eq.quantize_pack_table4(x, m, "fp16", out=out, status=st, check=False)
    torch.cuda.synchronize()
    print(w, "ok", st.item())
