#!/bin/bash
# A/B of compile-time variants on one box: AB_VARS="name|-DFOO=1;name2|-DFOO=2" (each built in a
# copy of the working tree under /tmp), AB_ARGS = bench args, AB_REPS repetitions (interleaved)
IFS=';' read -ra VS <<< "$AB_VARS"
for v in "${VS[@]}"; do
  IFS='|' read -r name flags <<< "$v"
  rm -rf /tmp/abv_$name; mkdir -p /tmp/abv_$name
  tar --exclude=./gpurun_out --exclude=./ab_old --exclude=./.git -cf - . | tar -xf - -C /tmp/abv_$name
  (cd /tmp/abv_$name && TIDE_NVCC_EXTRA="$flags" python -c "from paper_2605_20179_b200 import _build; _build.build(force=True)" > /dev/null 2>&1; echo "build $name rc=$?")
done
for rep in $(seq 1 ${AB_REPS:-3}); do
  for v in "${VS[@]}"; do
    IFS='|' read -r name flags <<< "$v"
    (cd /tmp/abv_$name && timeout 600 python bench.py --no-cpu --no-e2e --no-sub $AB_ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('us_per_layer_step'))")
  done
done
