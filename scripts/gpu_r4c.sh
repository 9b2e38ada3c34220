# plane-merged L1 dgrad A/B, interleaved: in-step (bench cfg2) and standalone, 3 rounds each
T=${1:-r4c}
mkdir -p gpurun_out
for i in 1 2 3; do for pm in 1 0; do
  DP_CONV_PM=$pm timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/${T}_b_${pm}_$i.json
  echo "PM=$pm $(DP_CONV_PM=$pm timeout 120 python scripts/conv_time.py dgrad 16 32 2>&1 | tail -1)" >> gpurun_out/${T}_time.log
done; done
cat gpurun_out/${T}_time.log
python - <<PY
import json
for i in (1, 2, 3):
    for pm in ("1", "0"):
        d = json.loads(open(f"gpurun_out/${T}_b_{pm}_{i}.json").read())
        print(i, pm, round(d["ms_per_step"], 4), d["clocks"]["sm_mhz"], {k: round(v["avg_ms"], 4) for k, v in d["kernels"].items() if "16" in k})
PY
