# coalesced bf16 conv epilogue (16x128b drain + permuted B columns): full GPU suite + cfg2/cfg4 bench + cfg2 ncu
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err
timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_cfg4.json 2> gpurun_out/r2l_cfg4.err
bash scripts/gpu_profile_conv.sh r2l
tail -5 gpurun_out/r2l_tests.log; python - <<'PY'
import json
for f in ("gpurun_out/r2l_bench.json", "gpurun_out/r2l_cfg4.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d["kernels"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
