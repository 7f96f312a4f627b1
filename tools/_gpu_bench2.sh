python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python bench.py > gpurun_out/bench_mini.json 2> gpurun_out/bench_mini.err; echo mini rc=$?
timeout 900 python bench.py --config sweep --steps 100 --warmup 10 --no-cpu > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo sweep rc=$?
timeout 900 python bench.py --config sweep --routing uniform --steps 100 --warmup 10 --no-cpu > gpurun_out/bench_sweep_uniform.json 2> gpurun_out/bench_sweep_uniform.err; echo sweepu rc=$?
timeout 900 python bench.py --routing uniform --steps 100 --warmup 10 --no-cpu > gpurun_out/bench_mini_uniform.json 2> gpurun_out/bench_mini_uniform.err; echo miniu rc=$?
timeout 900 python bench.py --config flash1 --steps 64 --warmup 8 --no-cpu > gpurun_out/bench_flash_8layers.json 2> gpurun_out/bench_flash.err; echo flash rc=$?
python - <<'PY'
import json
for f in ("mini","sweep","sweep_uniform","mini_uniform","flash_8layers"):
    try:
        d=json.load(open(f"gpurun_out/bench_{f}.json"))
    except Exception as e:
        print(f, "ERR", e); continue
    r=d["roofline"]
    print(f, d["value"], "ms/step", d["ms_per_step"], "ffn", r["achieved"], r["frac"], r["avg_launch_us"], "U", r["unique_experts_per_layer_step"], "e2e", d["e2e"]["value"] if d["e2e"] else None, d["clocks"], d["step_split"])
PY
