"""Summarise the GREEDY kernel SASS of a built library: hot-loop block size and local-memory traffic.
usage: python tools/sass_summary.py lib.so [kernel-substring]"""
import re, subprocess, sys
from collections import Counter
lib = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else "k_greedyILi1ELi64ELb1"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    L = [re.sub(r"/\*.*?\*/", "", l).strip().rstrip(";").strip() for l in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
    op = lambda l: l.split()[1] if l.startswith("@") else l.split()[0]
    blocks, cur = [], []
    for i, l in enumerate(L):
        cur.append(i)
        if "BRA" in l or "EXIT" in l:
            blocks.append(cur); cur = []
    print(name, len(L), "instrs")
    for b in blocks:
        c = Counter(op(L[i]) for i in b)
        if c["FFMA2.RM"] >= 8 or c["LDL"] + c["STL"] + c["LDL.LU"] > 0:
            print(f"  [{b[0]:5d},{b[-1]:5d}] n={len(b):4d} rm={c['FFMA2.RM']:3d} fsel={c['FSEL']:3d} "
                  f"ldl={c['LDL']+c['LDL.LU']+c['LDL.64']} stl={c['STL']+c['STL.64']} s2r={c['S2R']}")
