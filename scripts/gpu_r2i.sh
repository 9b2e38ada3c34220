# ring extension + global-row ring alignment: bitwise sharding invariance + conv parity + bench
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_kernels.py tests/test_gpu_tc_sharded.py tests/test_gpu_sharded.py tests/test_gpu_fullsize_oracle.py -q -x > gpurun_out/r2i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_cfg4.json 2> gpurun_out/r2i_cfg4.err
tail -5 gpurun_out/r2i_tests.log; python - <<'PY'
import json
for f in ("gpurun_out/r2i_bench.json", "gpurun_out/r2i_cfg4.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
