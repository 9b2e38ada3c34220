# plane-merged L1 dgrad: conv parity + the PM/two-ring bitwise A/B, then timings A/B
T=${1:-r4b}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "conv_tc or plane_merged or issue_paths or dense_conv" > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
for pm in 1 0 1 0; do echo "PM=$pm $(DP_CONV_PM=$pm timeout 120 python scripts/conv_time.py dgrad 16 32 2>&1 | tail -1)"; done > gpurun_out/${T}_time.log
for pm in 1 0; do DP_CONV_PM=$pm timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_cfg2_pm$pm.json 2> gpurun_out/${T}_cfg2_pm$pm.err; done
tail -2 gpurun_out/${T}_tests.log; cat gpurun_out/${T}_time.log
python - <<PY
import json
for pm in ("1", "0"):
    try:
        d = json.loads(open(f"gpurun_out/${T}_cfg2_pm{pm}.json").read().strip().splitlines()[-1])
        print(pm, d["ms_per_step"], {k: round(v["avg_ms"], 4) for k, v in d["kernels"].items()})
    except Exception as e:
        print(pm, "ERR", e)
PY
