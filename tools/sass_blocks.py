"""Group an ncu source page (SASS view) into straight-line blocks by execution count and list
the heaviest ones: instruction share, stall-sample share, first/last instruction.
  ncu -i rep.ncu-rep --page source --csv --print-source sass > x.csv
  python tools/sass_blocks.py x.csv "title" [top]"""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
h = rows[1]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
ins = [(r[1].strip(), int(r[iS]), int(r[iE])) for r in rows[2:] if len(r) > iE]
ts, ti = sum(x[1] for x in ins) or 1, sum(x[2] for x in ins) or 1
blocks = []
for i, (txt, smp, ex) in enumerate(ins):
    if blocks and blocks[-1]["e"] == ex:
        b = blocks[-1]; b["n"] += 1; b["s"] += smp; b["end"] = i
    else:
        blocks.append(dict(start=i, end=i, e=ex, n=1, s=smp))
print(f"# {title}")
print(f"# {len(ins)} SASS instructions, {ti} warp-instructions executed, {ts} stall samples")
print("# block            n_instr   executions  inst_share  sample_share  first .. last instruction")
for b in sorted(blocks, key=lambda b: -b["e"] * b["n"])[:top]:
    print(f"[{b['start']:5}-{b['end']:5}] {b['n']:6} {b['e']:12} {100*b['e']*b['n']/ti:9.1f}% {100*b['s']/ts:10.1f}%   "
          f"{ins[b['start']][0][:38]} .. {ins[b['end']][0][:38]}")
