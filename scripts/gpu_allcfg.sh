for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for c in cfg1 cfg3 cfg4 cfg5; do python - <<PY
import json
d=json.loads(open("gpurun_out/bench_$c.json").read().strip().splitlines()[-1])
print("$c", d["ms_per_step"], d.get("roofline",{}).get("kernel"), round(d.get("roofline",{}).get("frac",0),3), d.get("kernels"))
PY
done
