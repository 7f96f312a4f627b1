python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
export TIDE_BENCH_SAME_DEVICE=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --layers 2 --steps 4 --warmup 3 --no-cpu > gpurun_out/mp_replicas.json 2> gpurun_out/mp_replicas.err; echo replicas rc=$?
cut -c1-300 gpurun_out/mp_replicas.json; tail -3 gpurun_out/mp_replicas.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --ep --p2p --layers 2 --steps 4 --warmup 3 --no-cpu > gpurun_out/mp_ep.json 2> gpurun_out/mp_ep.err; echo ep rc=$?
cut -c1-400 gpurun_out/mp_ep.json; tail -3 gpurun_out/mp_ep.err
