#!/bin/bash
# ncu --set full capture of one kernel (regex) of one config: report copied to gpurun_out/
#   bash tools/prof1.sh c5 tc tc_pass1 tag
CFG=$1; PREC=$2; K=$3; TAG=${4:-x}
mkdir -p gpurun_out
python tools/run_eval.py --config $CFG --precision $PREC --iters 1 > gpurun_out/plain_$TAG.log 2>&1 || { cat gpurun_out/plain_$TAG.log; exit 1; }
ncu -f --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python tools/run_eval.py --config $CFG --precision $PREC --iters 2 > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
python3 tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep > gpurun_out/sum_$TAG.txt 2>&1
python3 tools/sass_hot.py gpurun_out/prof_$TAG.ncu-rep "$K" 40 > gpurun_out/sass_$TAG.txt 2>&1
head -30 gpurun_out/sum_$TAG.txt
