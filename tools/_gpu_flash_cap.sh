# BASELINE configs[2]: flash-shaped stack, capacity-limited with pinned-host refresh (8 layers:
# 51 GB of pinned host master), one block (T=32 steps), interval 4
free -g | head -2
for cap in 32 64 128 217; do
  timeout 1500 python bench.py --config flash1 --layers 8 --capacity $cap --interval 4 --steps 32 --warmup 4 --cpu-seconds 8 > gpurun_out/bench_flash_c$cap.json 2> gpurun_out/bench_flash_c$cap.err; echo "cap $cap rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_flash_c$cap.json')); print('flash C=$cap', d['value'], d['ms_per_step'], d['io'], d['step_split'], d['e2e']['value'] if d['e2e'] else None)"
  tail -2 gpurun_out/bench_flash_c$cap.err
done
