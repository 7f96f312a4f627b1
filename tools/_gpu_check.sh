# one GPU call: tests, smoke, default bench, launch list of the same command, ncu full of FFN + route
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_mini.json 2> gpurun_out/bench_mini.err; echo bench rc=$?; cut -c1-400 gpurun_out/bench_mini.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference.json 2>&1; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tide --csv --log-file gpurun_out/launches_mini_graph.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches.log 2>&1; echo ncu-launch rc=$?
python tools/launches.py gpurun_out/launches_mini_graph.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tide_ffn -s 60 -c 1 -o gpurun_out/ffn_full python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_ffn.log 2>&1; echo ncu-ffn rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tide_route -s 60 -c 1 -o gpurun_out/route_full python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_route.log 2>&1; echo ncu-route rc=$?
