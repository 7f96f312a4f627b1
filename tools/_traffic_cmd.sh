set -x
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for c in mini:640 sweep:640 flash1:256; do
  cfg=${c%%:*}; n=${c##*:}
  timeout 900 ncu --metrics $M --print-units base --clock-control none -k regex:tide_ffn -c $n --csv \
    --log-file gpurun_out/ffn_$cfg.csv python tools/ffn_traffic.py --config $cfg --algo gpurun_out/ffn_${cfg}_algo.json > gpurun_out/ffn_$cfg.log 2>&1
  echo "$cfg rc=$?"; tail -2 gpurun_out/ffn_$cfg.log
  python tools/ffn_traffic.py --config $cfg --join gpurun_out/ffn_$cfg.csv --algo gpurun_out/ffn_${cfg}_algo.json
done
cp profiles/ffn_traffic.json gpurun_out/ffn_traffic.json
