import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np, oracle, paper_1911_02079_b200 as eq
from sls_cases import sls_cases
for n,(packed, rows, d, aux, idx, ln, want) in enumerate(sls_cases()):
    if n != 1: continue
    p = eq.PackedTable4(rows, d, aux, buffer=packed)
    print(rows, d, aux, idx, ln)
    for r in range(rows):
        got = eq.sparse_lengths_sum_4bit(p, eq.PooledQuery([r], [1]))
        o,_,_ = oracle.sparse_lengths_sum4(packed, rows, d, aux, [r], [1])
        print(r, np.array_equal(got, o), got[0][:4], o[0][:4])
    got = eq.sparse_lengths_sum_4bit(p, eq.PooledQuery(idx, ln))
    print((got.view(np.uint32).astype(np.int64) - want.view(np.uint32)).tolist())
    stride = (d+1)//2 + 8
    B = packed.reshape(rows, stride)
    sc = B[:, 8:12].copy().view(np.float32); bi = B[:, 12:16].copy().view(np.float32)
    print(sc.ravel(), bi.ravel())
