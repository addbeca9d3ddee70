#!/bin/bash
# round-2 re-entry: GPU tests (incl. the reference's own suites through the drop-in), c5 tc profile
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02d_pytest.txt 2>&1
echo "pytest rc=$?"; tail -8 gpurun_out/r02d_pytest.txt
bash tools/profile_round.sh c5 tc r02d > gpurun_out/r02d_profile.log 2>&1
echo "profile rc=$?"
cat gpurun_out/r02d_c5_tc_ncu_summary.txt | head -80
cat gpurun_out/r02d_c5_tc_ncu_raw_key.txt
rm -f gpurun_out/*.ncu-rep.tmp
