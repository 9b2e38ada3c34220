# conv epilogue: per-unit addressing, division-free drain counters (+ coalesced drain)
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tc_sharded.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py tests/test_gpu_procs.py -q -x > gpurun_out/r2m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2m_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_cfg4.json 2> gpurun_out/r2m_cfg4.err
bash scripts/gpu_profile_conv.sh r2m
tail -3 gpurun_out/r2m_tests.log; python - <<'PY'
import json
for f in ("gpurun_out/r2m_bench.json", "gpurun_out/r2m_cfg4.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["clocks"]["sm_mhz"], {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
