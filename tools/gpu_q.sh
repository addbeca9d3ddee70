#!/bin/bash
# quick: per-kernel times of configs (ktime) [+ tc tests when $1 == t]
mkdir -p gpurun_out
for c in ${CFGS:-c5 c3 c4 c2}; do timeout 300 python tools/ktime.py $c ${PREC:-tc} 3 2>&1 | tail -1; done
if [ "$1" == "t" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "${TK:-tc}" 2>&1 | tail -4; fi
