"""Random row-gather reference points on this GPU (development probe): torch index_select of
36/40/128-byte rows vs the pooled-lookup kernel, timed inside a CUDA graph (no host gaps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_02079_b200 as eq


def graph_time(fn, n=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n


rows, nq = 20_000_000, 1 << 20
skip_torch = os.environ.get("SKIP_TORCH")
gen = torch.Generator(device="cuda").manual_seed(1)
idx = torch.randint(0, rows, (nq,), device="cuda", generator=gen)
for words in (() if skip_torch else (9, 10)):
    t = torch.randint(0, 1 << 30, (rows, words), dtype=torch.int32, device="cuda")
    ms = graph_time(lambda: torch.index_select(t, 0, idx))
    print(f"index_select {words*4} B rows: {ms*1e3:.1f} us  {nq/ms/1e6:.2f} G rows/s", flush=True)
    del t
for aux in ("fp16", "fp32"):
    x = torch.randn(rows, 64, device="cuda")
    p, _ = eq.quantize_pack_table4(x, "asym", aux)
    del x
    for batch, pool in ((16384, 64), (65536, 16), (1024, 1024)):
        ii = idx[: batch * pool]
        ln = torch.full((batch,), pool, dtype=torch.int64, device="cuda")
        q = eq.PooledQuery(ii, ln)
        out = torch.empty(batch, 64, device="cuda")
        ms = graph_time(lambda: eq.sparse_lengths_sum_4bit(p, q, out=out, check=False))
        print(f"sls 20Mx64 {aux} batch {batch} pool {pool}: {ms*1e3:.1f} us  "
              f"{batch*pool/ms/1e6:.2f} G rows/s", flush=True)
