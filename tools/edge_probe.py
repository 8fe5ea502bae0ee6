import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1911_02079_b200 as eq
f = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "edge.npz"))
meta = json.loads(str(f["meta"]))
start = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for k, m in enumerate(meta):
    if k < start: continue
    x = f[f"x_{k}"]
    for method in ("asym", "greedy"):
        print(k, m["name"], x.shape, method, flush=True, end=" ")
        t = time.time()
        try:
            p, rr = eq.quantize_pack_table4(torch.from_numpy(x).cuda(), method, "fp16", m["b"], m["r"], with_rows=True)
            torch.cuda.synchronize()
            ok = (m["greedy_error"] is None or method == "asym") and np.array_equal(p.buffer, f[f"{method}_fp16_{k}"])
            print("ok" if ok else "MISMATCH", f"{time.time()-t:.2f}s", flush=True)
        except ValueError as e:
            print("ValueError", e, flush=True)
