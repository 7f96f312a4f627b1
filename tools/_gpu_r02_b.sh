#!/bin/bash
# round 2: compute-sanitizer over the small cases, the NEXT-2 tau x C sweep with both models,
# route / FFN phase traces at the headline shape (one B200)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
bash tools/_gpu_sanitize.sh
mkdir -p gpurun_out/r02
timeout 1500 python tools/sweep_interval.py --layers 2 --out gpurun_out/r02/sweep_interval.json > gpurun_out/r02/sweep_interval.log 2>&1; echo sweep rc=$?
tail -30 gpurun_out/r02/sweep_interval.log
timeout 300 python tools/route_trace.py mini > gpurun_out/r02/route_trace_mini.txt 2>&1; echo rtrace rc=$?
cat gpurun_out/r02/route_trace_mini.txt | tail -20
