import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from oracle import rng
import paper_1911_02079_b200 as eq
x = rng.sample_table("gaussian", 0.0, 1.0, 1911, 64, 64)
want = oracle.quantize_pack_table(x, "greedy", 200, 0.16, "fp16")
p, rr = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "greedy", "fp16", with_rows=True)
lo, hi, it, i1 = [t.cpu().numpy() for t in (rr.xmin, rr.xmax, rr.info0, rr.info1)]
buf = p.buffer.reshape(-1, 36); wb = want.packed.reshape(-1, 36)
for i in range(12):
    print(i, lo[i], want.xmin[i], hi[i], want.xmax[i], it[i], want.info0[i], i1[i] >> 16, i1[i] & 0xffff, want.info1[i],
          np.nonzero(buf[i] != wb[i])[0].tolist(), buf[i][32:].tolist(), wb[i][32:].tolist())
pa, rra = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), "asym", "fp16", with_rows=True)
wa = oracle.quantize_pack_table(x, "asym", aux="fp16")
print("asym mismatching rows", np.nonzero((pa.buffer.reshape(-1,36) != wa.packed.reshape(-1,36)).any(1))[0][:20])
print(pa.buffer.reshape(-1,36)[0].tolist()); print(wa.packed.reshape(-1,36)[0].tolist())
