python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_ep_p2p.py tests/test_gpu_ep.py tests/test_gpu_parity.py -q 2>&1 | tail -5
timeout 600 python bench.py --ep --p2p --no-cpu > gpurun_out/bench_ep_p2p_world1.json 2> gpurun_out/bench_ep_p2p.err; echo bench-p2p rc=$?
timeout 600 python bench.py --ep --no-cpu 2>gpurun_out/bench_ep.err | grep '^{' > gpurun_out/bench_ep_world1.json; echo bench-ep rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/bench_ep_p2p_world1.json","gpurun_out/bench_ep_world1.json"):
    d=json.load(open(f)); print(f, d["value"], d["config"]["launch"], d["phases_us_per_layer_step"], d["roofline"]["frac"], d["e2e"]["value"])
PY
