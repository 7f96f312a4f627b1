python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in "" 1; do
  TIDE_ROUTER_NOCLUSTER=$v timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('nocluster=$v bench', d['value'], d['roofline']['frac'], d['phases_us_per_layer_step'])"
done
timeout 300 python tools/timeline.py mini 16 | head -12
