#!/bin/bash
# quick parity gate on the working tree, then the mini and sweep A/B against ab_old (a worktree)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py -x -q 2>&1 | tail -2
AB_ARGS="--no-sub" bash tools/_gpu_ab.sh 2>&1 | grep -v "build rc"
echo "== sweep"
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1)
for rep in 1 2; do for side in old new; do
  if [ $side = old ]; then D=ab_old; else D=.; fi
  (cd $D && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --config sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$side', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])")
done; done
