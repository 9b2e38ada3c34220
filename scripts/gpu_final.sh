# final measurement set: GPU suite, smoke, every config's bench line (+ sustained cfg2), the reference
# arm, launch lists + ncu --set full summaries (summarised on the box; .ncu-rep files dropped)
T=${1:-r3f}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python scripts/smoke_launches.py > gpurun_out/${T}_smoke_launches.txt 2>&1
timeout 600 python bench.py > gpurun_out/${T}_cfg2.json 2> gpurun_out/${T}_cfg2.err
for c in cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_$c.json 2> gpurun_out/${T}_$c.err; done
timeout 600 python bench.py --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_cfg2_sustained.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
bash scripts/gpu_r3b.sh ${T}
grep -E "passed|failed" gpurun_out/${T}_tests.log | tail -2
python - <<PY
import json
for f in ("cfg2", "cfg2_sustained", "cfg1", "cfg3", "cfg4", "cfg5", "ref"):
    try:
        d = json.loads(open(f"gpurun_out/${T}_{f}.json").read().strip().splitlines()[-1])
        print(f, d.get("ms_per_step"), d.get("value"), d.get("clocks", {}).get("sm_mhz"), d.get("roofline") and d["roofline"].get("frac"),
              {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d.get("kernels", {}).items()})
    except Exception as e:
        print(f, "ERR", e)
PY
