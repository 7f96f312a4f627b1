#!/bin/bash
# round 2 call D: NEXT-2 replay model on the GPU (copies exact vs measured) and the sweep with it
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_next.py -q -x 2>&1 | tail -3
mkdir -p gpurun_out/r02
timeout 2400 python tools/sweep_interval.py --layers 2 --out gpurun_out/r02/sweep_interval.json > gpurun_out/r02/sweep_interval.log 2>&1; echo sweep rc=$?
