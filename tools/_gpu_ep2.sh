python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_ep_p2p.py tests/test_gpu_ep.py -q 2>&1 | tail -3
timeout 600 python bench.py --ep --p2p --no-cpu > gpurun_out/bench_ep_p2p_world1.json 2> gpurun_out/bench_ep_p2p.err; echo bench-p2p rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_ep_p2p_world1.json')); print(d['value'], d['phases_us_per_layer_step'], d['roofline']['frac'], d['e2e']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tide --csv --log-file gpurun_out/launches_ep_p2p.csv python bench.py --ep --p2p --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches_ep.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/launches_ep_p2p.csv
