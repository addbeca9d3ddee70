#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-sw}
timeout 300 python tools/ktime.py c5 tc 3 > gpurun_out/${TAG}_kt.txt 2>&1; echo "ktime rc=$?"; tail -5 gpurun_out/${TAG}_kt.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "tc" > gpurun_out/${TAG}_pytest.txt 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/${TAG}_pytest.txt
bash tools/quick.sh "" "c5:tc c3:tc c4:tc c2:tc" 2>&1
PGX_TC_SWEEP=0 bash tools/quick.sh "" "c5:tc" 2>&1
