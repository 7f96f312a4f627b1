python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -x -q --tb=short 2>&1 | tail -4
for rep in 1 2; do
  for v in "" 1; do
    TIDE_FFN_NOFUSE=$v timeout 600 python bench.py --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('nofuse=$v', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])"
  done
done
