set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests/test_gpu_ep_p2p.py -x -q -k "not two_processes" > gpurun_out/pytest_p2p.log 2>&1; echo p2p rc=$?; tail -30 gpurun_out/pytest_p2p.log
timeout 300 python -m pytest tests/test_gpu_ep_p2p.py -x -q -k "two_processes" > gpurun_out/pytest_p2p_ipc.log 2>&1; echo ipc rc=$?; tail -30 gpurun_out/pytest_p2p_ipc.log
timeout 600 python bench.py --ep --p2p --no-cpu > gpurun_out/bench_ep_p2p_world1.json 2> gpurun_out/bench_ep_p2p.err; echo bench-p2p rc=$?; cut -c1-300 gpurun_out/bench_ep_p2p_world1.json; tail -3 gpurun_out/bench_ep_p2p.err
timeout 600 python bench.py --ep --no-cpu > gpurun_out/bench_ep_world1.json 2> gpurun_out/bench_ep.err; echo bench-ep rc=$?; cut -c1-300 gpurun_out/bench_ep_world1.json
