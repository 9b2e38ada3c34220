# round-2 re-entry: full GPU suite + smoke + all-config bench lines + cfg2 launch list / ncu
set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2k_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
for c in cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_$c.json 2> gpurun_out/r2k_$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2k_ref.json 2> gpurun_out/r2k_ref.err
bash scripts/gpu_profile_conv.sh r2k
tail -5 gpurun_out/r2k_tests.log; cat gpurun_out/r2k_smoke.log | tail -3
python - <<'PY'
import json
for f in ("r2k_bench", "r2k_cfg1", "r2k_cfg3", "r2k_cfg4", "r2k_cfg5", "r2k_ref"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, d.get("ms_per_step"), d.get("value"), d.get("roofline", {}).get("frac"), {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d.get("kernels", {}).items()})
    except Exception as e:
        print(f, "ERR", e)
PY
