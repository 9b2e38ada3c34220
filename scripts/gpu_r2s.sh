# SS wgrad: single staged dY copy (overlapping MN atoms, LBO = one row) + two-level reduce; full GPU suite, cfg4 bench, cfg4 launch list
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2s_tests.log
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2s_cfg4.json 2> gpurun_out/r2s_cfg4.err
DP_WGRAD_SDY=0 timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2s_cfg4_nosdy.json 2> gpurun_out/r2s_cfg4_nosdy.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv \
    --log-file gpurun_out/r2s_cfg4_launches.csv python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
grep -E "passed|failed" gpurun_out/r2s_tests.log | tail -3; tail -1 gpurun_out/r2s_tests.log
python - <<'PY'
import json
for f in ("gpurun_out/r2s_cfg4.json", "gpurun_out/r2s_cfg4_nosdy.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["clocks"]["sm_mhz"], {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
python scripts/ncu_summary.py launches gpurun_out/r2s_cfg4_launches.csv gpurun_out/r2s_cfg4_launches.md > /dev/null; cat gpurun_out/r2s_cfg4_launches.md
