# refresh of every committed bench line / profile at HEAD (one B200)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv,noheader
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | cut -c1-120
run() { name=$1; shift; timeout 1200 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_$name.json') if l.startswith('{')][0]); r=d['roofline']; print('  ', d['value'], 'frac', r['frac'], 'e2e', (d['e2e'] or {}).get('value'), 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" 2>/dev/null; }
run mini
run mini_uniform --routing uniform --steps 100 --warmup 10 --no-cpu
run sweep --config sweep --steps 100 --warmup 10 --no-cpu
run sweep_uniform --config sweep --routing uniform --steps 100 --warmup 10 --no-cpu
run flash_8layers --config flash1 --steps 64 --warmup 8 --no-cpu
run ep_world1 --ep --no-cpu
run ep_p2p_world1 --ep --p2p --no-cpu
run capacity128_4layers --layers 4 --capacity 128 --steps 32 --warmup 4 --no-cpu
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>&1; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tide --csv --log-file gpurun_out/launches_mini_graph.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tide_ffn -s 60 -c 1 -o gpurun_out/ffn_full python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu-ffn rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tide --csv --log-file gpurun_out/launches_ep_p2p.csv python bench.py --ep --p2p --steps 4 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu-ep rc=$?
