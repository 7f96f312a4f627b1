echo "== TC router"; timeout 300 python tools/router_err.py
echo "== CC router"; TIDE_ROUTER_CC=1 timeout 300 python tools/router_err.py
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/timeline.py mini 16 2>&1 | tail -5
for cc in 0 1; do for cfg in mini sweep; do
  if [ $cc = 1 ]; then export TIDE_ROUTER_CC=1; else unset TIDE_ROUTER_CC; fi
  timeout 600 python bench.py --config $cfg --steps 96 --warmup 32 --no-cpu --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('cc=$cc $cfg', d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_us_per_layer_step']['router_ms'])"
done; done
