#!/bin/bash
# A/B timing of library variants, interleaved: tools/ab.sh "case ..." lib1 lib2 ...
# ("" = the in-tree build).  Run on the GPU box.
cases=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    echo "== ${v:-tree}"
    EQ4_LIB=$v python tools/probe_perf.py $cases 2>&1 | grep -E "^(greedy|asym|hist)"
  done
done
