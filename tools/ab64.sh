#!/bin/bash
# A/B of variant builds on the fp64 grid path: bash tools/ab64.sh "c2 c4" v1 v2 ...
CFGS=$1; shift
for v in "$@"; do
  for c in $CFGS; do
    PGX_LIB=paper_2605_20816_b200/lib/var/$v.so timeout 300 python tools/ktime.py $c fp64 5 | sed "s/^/$v /"
  done
done
