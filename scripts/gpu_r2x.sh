# power / clock under the cfg2 step: short and long timed regions
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2x_s20.json 2>/dev/null
timeout 600 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/r2x_s300.json 2>/dev/null
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2x_cfg3.json 2>/dev/null
python - <<'PY'
import json
for f in ("r2x_s20", "r2x_s300", "r2x_cfg3"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, round(d["ms_per_step"], 4), d["clocks"], {k: round(v["avg_ms"], 4) for k, v in d["kernels"].items()})
PY
nvidia-smi -q -d POWER,CLOCK | head -60
