#!/bin/bash
export AB_VARS="p0|;p4|-DTIDE_FFN_PFD=4;p8|-DTIDE_FFN_PFD=8;p16|-DTIDE_FFN_PFD=16"
AB_REPS=3 bash tools/_gpu_ab_vars.sh
echo "== sweep"
for rep in 1 2; do for name in p0 p4 p8 p16; do
  (cd /tmp/abv_$name && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --config sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('us_per_layer_step'))")
done; done
echo "== flash1 8 layers"
for rep in 1 2; do for name in p0 p8; do
  (cd /tmp/abv_$name && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --config flash1 --layers 8 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('us_per_layer_step'))")
done; done
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
