set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k sweep_uniform > gpurun_out/pytest_new.log 2>&1; echo new rc=$?; tail -3 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_mini.json 2> gpurun_out/bench_mini.err; echo bench rc=$?; cut -c1-300 gpurun_out/bench_mini.json
