"""Device timing of the pooled lookup (development probe): rows:d:aux:batch:pooling cases."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq

cases = sys.argv[1:] or ["20000000:64:fp16:16384:64", "20000000:64:fp32:16384:64"]
for c in cases:
    rows, d, aux, batch, pool = c.split(":")
    rows, d, batch, pool = int(rows), int(d), int(batch), int(pool)
    x = torch.randn(rows, d, device="cuda")
    p, _ = eq.quantize_pack_table4(x, "asym", aux)
    del x
    g = torch.Generator(device="cuda").manual_seed(1)
    idx = torch.randint(0, rows, (batch * pool,), device="cuda", generator=g)
    ln = torch.full((batch,), pool, dtype=torch.int64, device="cuda")
    q = eq.PooledQuery(idx, ln)
    out = torch.empty(batch, d, device="cuda")
    f = lambda: eq.sparse_lengths_sum_4bit(p, q, out=out, check=False)
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 20
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    alg = batch * pool * (eq.bytes_per_pooled_row("int4", d, aux) + 8) + batch * d * 4
    print(f"sls {c}: {ms*1e3:.1f} us  {batch*pool*d/ms/1e6:.1f} G sums/s  "
          f"{alg/ms/1e6:.1f} GB/s alg  {batch*pool/ms/1e6:.2f} G rows/s", flush=True)
