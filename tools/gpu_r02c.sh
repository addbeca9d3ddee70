#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_extensions_gpu.py tests/test_heuristics.py -m gpu -x -q 2>&1 | tail -15
bash tools/profile_round.sh c5 tc r02c > gpurun_out/r02c_profile.log 2>&1
echo "profile rc=$?"
rm -f gpurun_out/*.ncu-rep
