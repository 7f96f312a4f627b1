#!/bin/bash
# round-2 closing refresh at HEAD on one B200: GPU tests + smoke + every bench line, the profile set
# (launch lists, ncu full route/FFN, DRAM traffic joins, traces), sanitizers
bash tools/_gpu_final.sh > gpurun_out/final.log 2>&1
echo "== final"; tail -32 gpurun_out/final.log
bash tools/_gpu_profile_r02.sh > gpurun_out/profile.log 2>&1
echo "== profile"; tail -10 gpurun_out/profile.log | cut -c1-200
rm -f gpurun_out/sanitizer/summary.txt
bash tools/_gpu_sanitize.sh > /dev/null 2>&1
echo "== sanitizer"; cut -c1-150 gpurun_out/sanitizer/summary.txt
