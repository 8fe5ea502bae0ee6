"""One GREEDY launch on the bench table (for ncu captures): python tools/one_greedy.py [rows] [d] [dist]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dist = sys.argv[3] if len(sys.argv) > 3 else "mixed"
x = (workloads.mixed_table if dist == "mixed" else workloads.gaussian_table)(rows, d, 1911)
out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
eq.quantize_pack_table4(x, "greedy", "fp16", out=out, status=st, check=False)
torch.cuda.synchronize()
print("ok", int(st.item()))
