#!/bin/bash
# round 2 call E: EP list appends in the router (owner lists built by the sources) -- EP GPU
# tests, sanitizer of the peer-memory case, A/B vs ab_old
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo old build rc=$?)
timeout 900 python -m pytest tests/test_gpu_ep_p2p.py tests/test_gpu_ep.py tests/test_gpu_bench.py -q -x 2>&1 | tail -3
mkdir -p gpurun_out/sanitizer
bash tools/_gpu_sanitize.sh p2p_world2 > /dev/null 2>&1; tail -3 gpurun_out/sanitizer/summary.txt | cut -c1-150
for rep in 1 2 3; do
  for side in old new; do
    if [ $side = old ]; then D=ab_old; else D=.; fi
    (cd $D && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --ep --p2p 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ep-p2p $side', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('phases_us_per_layer_step'))")
  done
done
timeout 600 python bench.py --no-cpu --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('single', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d.get('phases_us_per_layer_step'))"
