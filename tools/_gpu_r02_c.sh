#!/bin/bash
# round 2 call C: EP early-trigger A/B (ab_old = previous HEAD), EP GPU tests, racecheck of the
# peer-memory case after the shared-flag fix, the warm/median tau x C sweep, route + layer timeline
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo old build rc=$?)
timeout 900 python -m pytest tests/test_gpu_ep_p2p.py tests/test_gpu_ep.py -q -x 2>&1 | tail -2
for rep in 1 2 3; do
  for side in old new; do
    if [ $side = old ]; then D=ab_old; else D=.; fi
    (cd $D && timeout 600 python bench.py --no-cpu --no-e2e --no-sub --ep --p2p 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ep-p2p $side', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])")
  done
done
timeout 600 python bench.py --no-cpu --no-e2e --no-sub 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('single', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])"
mkdir -p gpurun_out/sanitizer gpurun_out/r02
bash tools/_gpu_sanitize.sh p2p_world2 > /dev/null 2>&1; tail -3 gpurun_out/sanitizer/summary.txt
timeout 300 python tools/route_trace.py mini > gpurun_out/r02/route_trace_mini.txt 2>&1; echo rtrace rc=$?; cat gpurun_out/r02/route_trace_mini.txt
timeout 300 python tools/timeline.py mini > gpurun_out/r02/timeline_mini.txt 2>&1; echo timeline rc=$?; cat gpurun_out/r02/timeline_mini.txt
timeout 2400 python tools/sweep_interval.py --layers 2 --out gpurun_out/r02/sweep_interval.json > gpurun_out/r02/sweep_interval.log 2>&1; echo sweep rc=$?
