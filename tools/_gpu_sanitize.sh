#!/bin/bash
# compute-sanitizer over the small TIDE cases (tools/sanitize_cases.py); logs in
# gpurun_out/sanitizer/<tool>_<case>.txt, one summary line per run in summary.txt.
# usage (on the GPU box): bash tools/_gpu_sanitize.sh [cases...]
mkdir -p gpurun_out/sanitizer
CASES=${@:-toy_device_all toy_host_master bf16_tc graph_replay p2p_world2}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in $CASES; do
    log=gpurun_out/sanitizer/${tool}_${c}.txt
    start=$(date +%s)
    timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(( $(date +%s) - start ))s :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok$' $log | tr '\n' ' ')" >> gpurun_out/sanitizer/summary.txt
  done
done
cat gpurun_out/sanitizer/summary.txt
