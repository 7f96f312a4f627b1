python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_mini.json 2> gpurun_out/bench_mini.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_mini.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
timeout 600 python bench.py --ep --p2p --no-cpu > gpurun_out/bench_ep_p2p_world1.json 2> gpurun_out/bench_ep_p2p.err; echo bench-p2p rc=$?
timeout 600 python bench.py --ep --no-cpu 2>/dev/null | grep '^{' > gpurun_out/bench_ep_world1.json; echo bench-ep rc=$?
python -c "
import json
for f in ('bench_ep_p2p_world1','bench_ep_world1'):
    d=json.load(open(f'gpurun_out/{f}.json')); print(f, d['value'], d['roofline']['frac'], d['e2e']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tide --csv --log-file gpurun_out/launches_ep_p2p.csv python bench.py --ep --p2p --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches_ep.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/launches_ep_p2p.csv
