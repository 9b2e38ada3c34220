# RF flush groups (4 rows) in the bf16x3 wgrad: fp32 parity (incl. full cfg1 oracle), cfg1 bench; conv ablations on random dY
timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py tests/test_gpu_kernels.py tests/test_gpu_sharded.py -q > gpurun_out/r2z_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2z_tests.log
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2z_cfg1.json 2> gpurun_out/r2z_cfg1.err
for w in "fwd 16 32" "dgrad 16 32" "wgrad 16 32" "fwd 32 32" "dgrad 32 32" "wgrad 32 32"; do
  for d in 0 13; do DP_CONV_DBG=$d timeout 120 python scripts/conv_time.py $w; done
done > gpurun_out/r2z_abl.txt 2>&1
tail -2 gpurun_out/r2z_tests.log; cat gpurun_out/r2z_abl.txt
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2z_cfg1.json").read().strip().splitlines()[-1])
print("cfg1", d["ms_per_step"], {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d["kernels"].items()})
PY
