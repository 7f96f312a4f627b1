#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
AB_ARGS="--no-sub" bash tools/_gpu_ab.sh 2>&1 | grep -v "build rc"
echo "== ep p2p world 1"
for rep in 1 2; do for side in old new; do
  if [ $side = old ]; then D=ab_old; else D=.; fi
  (cd $D && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --ep --p2p 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$side', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])")
done; done
