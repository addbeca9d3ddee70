#!/bin/bash
# round state check (bash tools/gpu_round.sh TAG): GPU tests, smoke, default bench (c5 tc) + reference arm, c5 profile, quick lines
mkdir -p gpurun_out
TAG=${1:-r02f}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.txt 2>&1
echo "pytest rc=$?"; tail -6 gpurun_out/${TAG}_pytest.txt
python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1; tail -2 gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 400 gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_reference_bench.json 2> gpurun_out/${TAG}_reference_bench.err
echo "ref rc=$?"
bash tools/profile_round.sh c5 tc $TAG > gpurun_out/${TAG}_profile.log 2>&1
echo "profile rc=$?"
bash tools/quick.sh "" "c1:tc c2:tc c3:tc c4:tc paper140:tc"
for c in c1 c2 c3 c4 paper140; do cp gpurun_out/q_${c}_tc.json gpurun_out/${TAG}_${c}_tc_quick.json; done
rm -f gpurun_out/*.ncu-rep.tmp
