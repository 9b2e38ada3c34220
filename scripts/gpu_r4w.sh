# multi-rank sanity at the final build (r4w) on the one GPU (gloo-cuda, self-launched): every config completes, no CUDA-core routing
for c in cfg2 cfg1 cfg4 cfg5; do timeout 900 python bench.py --gpus 2 --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r4w_${c}_g2.json 2> gpurun_out/r4w_${c}_g2.err; echo "$c rc=$?"; done
timeout 900 python bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r4w_cfg2_g4.json 2> gpurun_out/r4w_cfg2_g4.err; echo "cfg2 g4 rc=$?"
timeout 900 python bench.py --gpus 2 --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r4w_cfg3_g2.json 2> gpurun_out/r4w_cfg3_g2.err; echo "cfg3 g2 rc=$?"
timeout 600 python -m pytest tests/test_gpu_procs.py tests/test_gpu_comm.py -q 2>&1 | tail -2
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r4w_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get("n_gpus"), round(d.get("ms_per_step"), 3), d.get("simt_calls"), d.get("gpu_launches_per_step"))
    except Exception as e:
        print(f, "ERR", e)
PY
