# float4 tile split kernel for the bf16x3 operands: bit-exact parts test, fp32 conv parity, cfg1 bench + launch list
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize_oracle.py tests/test_gpu_sharded.py -q > gpurun_out/r2r_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_tests.log
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2r_cfg1.json 2> gpurun_out/r2r_cfg1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv \
    --log-file gpurun_out/r2r_cfg1_launches.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
grep -E "passed|failed" gpurun_out/r2r_tests.log | tail -3; tail -1 gpurun_out/r2r_tests.log
python - <<'PY'
import json
for f in ("gpurun_out/r2r_cfg1.json",):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["clocks"]["sm_mhz"], {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
python scripts/ncu_summary.py launches gpurun_out/r2r_cfg1_launches.csv gpurun_out/r2r_cfg1_launches.md > /dev/null; cat gpurun_out/r2r_cfg1_launches.md
