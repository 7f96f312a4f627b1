#!/bin/bash
# Round-2 profile refresh on one B200 (run from the repo root under gpurun):
#   launch lists (ncu gpu__time_duration per launch) of the headline and the EP world-1 step,
#   ncu --set full captures of the route and FFN kernels (mini headline), the DRAM-traffic
#   join of every FFN launch of one block (profiles/ffn_traffic.json), the bench lines.
# Outputs land in gpurun_out/r02/; the committed summaries are made from them by
# tools/ncu_summary.py / tools/launches.py.
set -u
O=gpurun_out/r02
mkdir -p $O
NOSUB="--no-cpu --no-e2e --no-sub"
# launch list (serialised, cold caches): kernel shares of the graph-replayed step
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tide --csv \
  --log-file $O/launches_mini_graph.csv python bench.py --steps 4 --warmup 3 $NOSUB > /dev/null 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tide --csv \
  --log-file $O/launches_ep_p2p.csv python bench.py --ep --p2p --steps 4 --warmup 3 $NOSUB > /dev/null 2>&1
echo "ncu launches ep rc=$?"
# full captures (one launch each, past the warm-up)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tide_route -s 60 -c 1 \
  -o $O/route_full python bench.py --steps 4 --warmup 3 $NOSUB > /dev/null 2>&1
echo "ncu route rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tide_ffn -s 60 -c 1 \
  -o $O/ffn_full python bench.py --steps 4 --warmup 3 $NOSUB > /dev/null 2>&1
echo "ncu ffn rc=$?"
# DRAM traffic vs algorithmic bytes, every FFN launch of one block
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for c in mini:640 sweep:640 flash1:256; do
  cfg=${c%%:*}; n=${c##*:}
  timeout 900 ncu --metrics $M --print-units base --clock-control none -k regex:tide_ffn -c $n --csv \
    --log-file $O/ffn_$cfg.csv python tools/ffn_traffic.py --config $cfg --algo $O/ffn_${cfg}_algo.json > $O/ffn_$cfg.log 2>&1
  echo "$cfg rc=$?"
  python tools/ffn_traffic.py --config $cfg --join $O/ffn_$cfg.csv --algo $O/ffn_${cfg}_algo.json
done
cp profiles/ffn_traffic.json $O/ffn_traffic.json
# route / layer timelines and the FFN stream-rate timeline (kernel %globaltimer traces)
timeout 300 python tools/route_trace.py mini > $O/route_trace_mini.txt 2>&1
timeout 300 python tools/timeline.py mini > $O/timeline_mini.txt 2>&1
timeout 300 python tools/ffn_items.py mini 12 > $O/ffn_items_mini.txt 2>&1
echo traces rc=$?
