#!/bin/bash
# round-2 state check: GPU tests, default bench, reference arm, c5 tc profile, quick lines c1-c4
mkdir -p gpurun_out
bash tools/gpu_check.sh r02b
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b_reference_bench.json 2> gpurun_out/r02b_reference_bench.err
echo "ref rc=$?"; tail -c 600 gpurun_out/r02b_reference_bench.json
bash tools/profile_round.sh c5 tc r02b > gpurun_out/r02b_profile.log 2>&1
echo "profile rc=$?"
cat gpurun_out/r02b_c5_tc_ncu_summary.txt | head -60
bash tools/quick.sh "" "c1:tc c2:tc c3:tc c4:tc c5:fp64"
python __graft_entry__.py smoke > gpurun_out/r02b_smoke.txt 2>&1; tail -3 gpurun_out/r02b_smoke.txt
rm -f gpurun_out/*.ncu-rep.tmp
