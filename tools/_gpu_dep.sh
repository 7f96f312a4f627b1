python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
for d in 0 1 2; do
  echo "== dep_after $d"
  TIDE_FFN_DEP_AFTER=$d timeout 300 python tools/ffn_probe.py 2>&1 | head -2
  TIDE_FFN_DEP_AFTER=$d timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('bench', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])"
done
