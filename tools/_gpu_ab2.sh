#!/bin/bash
# A/B ab_old (reference checkout) vs the working tree: AB_ARGS_LIST="name|args;..." (3 reps)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo old build rc=$?)
if [ -n "$AB_TESTS" ]; then timeout 1200 python -m pytest $AB_TESTS -q -x 2>&1 | tail -2; fi
IFS=';' read -ra VS <<< "$AB_ARGS_LIST"
for rep in $(seq 1 ${AB_REPS:-3}); do
  for v in "${VS[@]}"; do
    IFS='|' read -r name args <<< "$v"
    for side in old new; do
      if [ $side = old ]; then D=ab_old; else D=.; fi
      (cd $D && timeout 600 python bench.py --no-cpu --no-e2e --no-sub $args 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name $side', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('us_per_layer_step'))")
    done
  done
done
