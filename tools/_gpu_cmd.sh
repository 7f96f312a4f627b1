timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/timeline.py mini 16 2>&1 | tail -14
timeout 600 python bench.py --steps 192 --warmup 32 --no-cpu --no-e2e --graph > gpurun_out/bench_graph.json 2>gpurun_out/bench_graph.err; python -c "
import json; d=json.load(open('gpurun_out/bench_graph.json')); print('graph', d['value'], d['ms_per_step'], d['roofline']['frac'], d['phases_us_per_layer_step'])"
