python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 300 python tools/ffn_items.py mini 12
timeout 300 python tools/ffn_probe.py
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('bench', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
