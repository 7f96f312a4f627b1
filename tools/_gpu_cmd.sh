timeout 300 python tools/router_err.py
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/timeline.py sweep 16 2>&1 | tail -4
for cfg in sweep mini; do
  timeout 600 python bench.py --config $cfg --steps 96 --warmup 32 --no-cpu --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('$cfg', d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_us_per_layer_step']['router_ms'])"
done
