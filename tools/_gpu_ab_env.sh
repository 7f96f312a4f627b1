#!/bin/bash
# A/B of env/arg variants of the working tree on one box: AB_VARIANTS="name|ENV=..|args;..."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
IFS=';' read -ra VS <<< "$AB_VARIANTS"
for rep in $(seq 1 ${AB_REPS:-3}); do
  for v in "${VS[@]}"; do
    IFS='|' read -r name envs args <<< "$v"
    env $envs timeout 600 python bench.py --no-cpu --no-e2e --no-sub $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('us_per_layer_step'))"
  done
done
