python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tide --csv --log-file gpurun_out/launches_ep_p2p.csv python bench.py --ep --p2p --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches_ep.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/launches_ep_p2p.csv
