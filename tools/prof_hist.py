"""One HIST-BRUTE launch (16,384 x 64 N(0,1), b=200) as an ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq
from paper_1911_02079_b200 import workloads
x = workloads.gaussian_table(16384, 64, 7)
for _ in range(2):
    eq.quantize_pack_table4(x, "hist-brute", "fp16", check=False)
torch.cuda.synchronize()
print("ok")
