import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from oracle import rng
import paper_1911_02079_b200 as eq
x = rng.sample_table("gaussian", 0.0, 1.0, 1911, 10000, 64)
want = oracle.quantize_pack_table(x, "greedy", 200, 0.16, "fp16")
p, rr = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "greedy", "fp16", with_rows=True)
lo, hi, it, i1 = [t.cpu().numpy() for t in (rr.xmin, rr.xmax, rr.info0, rr.info1)]
bad = np.nonzero((lo != want.xmin) | (hi != want.xmax))[0]
print("mismatching rows", len(bad), bad[:20])
for i in bad[:8]:
    g = oracle.clip_range_greedy(x[i])
    print(i, "ours", i1[i] >> 16, i1[i] & 0xffff, it[i], "ref", g.best_i, g.best_j, g.iters)
