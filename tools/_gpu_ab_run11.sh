#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
export AB_VARS="merge|;rounds|-DTIDE_ROUTE_MERGE=0"
AB_REPS=3 bash tools/_gpu_ab_vars.sh
echo "== sweep"
for rep in 1 2; do for name in merge rounds; do
  (cd /tmp/abv_$name && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --config sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('us_per_layer_step'))")
done; done
