"""Aggregate an ncu `--page source --print-source cuda,sass` CSV by CUDA source line.
  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv
  python tools/src_profile.py x.csv [top]
Prints per source line: share of stall samples, share of executed warp instructions."""
import csv, sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, agg, src = None, None, defaultdict(lambda: [0, 0]), {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] and r[0] != "-" and r[2] == "-":      # a source line row
        cur = (fname, int(r[0])); src[cur] = r[1][:80]; continue
    try:
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        ie = int(r[hdr.index("Instructions Executed")])
    except ValueError:
        continue
    key = (fname, int(r[0])) if r[0] not in ("", "-") else cur
    agg[key][0] += s; agg[key][1] += ie
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts}  total warp instructions {ti}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/ts:5.1f}% samp {100*v[1]/ti:5.1f}% inst  {k[0]}:{k[1]:<5} {src.get(k, '')}")
