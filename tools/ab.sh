#!/bin/bash
# A/B kernel variants built into paper_2605_20816_b200/lib/var/*.so:
#   bash tools/ab.sh "c2 c5" base other ...
CFGS=$1; shift
for v in "$@"; do
  for c in $CFGS; do
    PGX_LIB=paper_2605_20816_b200/lib/var/$v.so timeout 300 python tools/ktime.py $c tc 5 | sed "s/^/$v /"
  done
done
