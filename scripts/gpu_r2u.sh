# (1) TS wgrad junk-lane zeroing (power) A/B in the cfg2 step; (2) attention fwd exp2 MUFU/FMA split sweep
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2u_z$i.json 2>/dev/null
  DP_CONV_DBG=64 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2u_nz$i.json 2>/dev/null
done
for pl in 2 3 4 1; do DP_ATTN_POLY=$pl S=16384 timeout 300 python scripts/attn_time.py; done > gpurun_out/r2u_poly.txt 2>&1
for pl in 2 3; do DP_ATTN_POLY=$pl S=65536 timeout 300 python scripts/attn_time.py; done >> gpurun_out/r2u_poly.txt 2>&1
python - <<'PY'
import json
for f in ("z1", "nz1", "z2", "nz2"):
    try:
        d = json.loads(open(f"gpurun_out/r2u_{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"], {k: round(v["avg_ms"], 4) for k, v in d["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
cat gpurun_out/r2u_poly.txt
