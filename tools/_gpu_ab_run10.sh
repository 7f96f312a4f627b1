#!/bin/bash
export AB_VARS="base|;prew|-DTIDE_ROUTE_PREW=1"
AB_REPS=3 bash tools/_gpu_ab_vars.sh
echo "== sweep"
for rep in 1 2; do for name in base prew; do
  (cd /tmp/abv_$name && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --config sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('us_per_layer_step'))")
done; done
(cd /tmp/abv_prew && timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1)
