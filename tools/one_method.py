"""One launch of a method on a synthetic N(0,1) table (for ncu captures):
    python tools/one_method.py method rows d"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads
method, rows, d = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
x = workloads.gaussian_table(rows, d, 7)
out = torch.empty(rows * eq.packed_row_stride(d, "fp16"), dtype=torch.uint8, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
eq.quantize_pack_table4(x, method, "fp16", out=out, status=st, check=False)
torch.cuda.synchronize()
print("ok", int(st.item()))
