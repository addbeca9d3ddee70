#!/bin/bash
# round-2 first GPU call: probes + state check
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
timeout 300 ./tools/probe_r2 > gpurun_out/r02a_probe.txt 2>&1
echo "probe rc=$?"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.txt 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02a_pytest.txt
bash tools/quick.sh "" "c5:tc c5:fp64 c3:tc c4:tc c1:tc" 2>&1 | tee gpurun_out/r02a_quick.txt
cat gpurun_out/r02a_probe.txt
