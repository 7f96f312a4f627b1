#!/bin/bash
export AB_VARS="w32|;w64|-DTIDE_FFN_DEPW=64;w32f|-DTIDE_FFN_PFENCE=1;w64f|-DTIDE_FFN_DEPW=64 -DTIDE_FFN_PFENCE=1"
AB_REPS=3 bash tools/_gpu_ab_vars.sh
echo "== sweep"
for rep in 1 2; do for name in w32 w64 w32f w64f; do
  (cd /tmp/abv_$name && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --config sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('us_per_layer_step'))")
done; done
