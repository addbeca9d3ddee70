#!/bin/bash
# compute-sanitizer runs of the hand-written mbarrier / TMEM / bulk-copy kernels
# (tensor-core sweep, grad and assign; fp64 grid kernels; general kernels + tail).
# Summaries land in gpurun_out/sanitize_*.txt (copied to profiles/ per round).
# NOTE (round 2): compute-sanitizer is closed on this GPU pool (every tool exits 86 with the
# message kept in profiles/r02_sanitizer_closed_on_pool.txt); the script is kept for pools that allow it.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  for cfg in "c1 tc" "c2 tc" "c2 fp64" "c1 exact"; do
    set -- $cfg
    out=gpurun_out/sanitize_${tool}_$1_$2.txt
    timeout 900 $CS --tool $tool --print-limit 20 python tools/run_eval.py --config $1 --precision $2 --iters 1 --assign > $out 2>&1
    echo "$tool $1 $2 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out | tail -1)"
  done
done
# a padded (140 x 140) tensor-core problem under memcheck
timeout 900 $CS --tool memcheck --print-limit 20 python tools/run_eval.py --config paper140 --precision tc --iters 1 --assign > gpurun_out/sanitize_memcheck_paper140_tc.txt 2>&1
echo "memcheck paper140 tc rc=$? $(grep -E 'ERROR SUMMARY' gpurun_out/sanitize_memcheck_paper140_tc.txt | tail -1)"
